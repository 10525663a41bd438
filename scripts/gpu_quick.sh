# quick GPU iteration: parity (small/medium) + per-kernel times and event counters
mkdir -p gpurun_out
T=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python scripts/stats.py ${CFGS:-c2 c3 c4 c5} > gpurun_out/${T}_stats.log 2>&1
