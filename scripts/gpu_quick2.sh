# quick: all GPU tests (not the full O1), per-kernel times + stats, bench c5
mkdir -p gpurun_out
T=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python scripts/stats.py ${CFGS:-c4 c5} > gpurun_out/${T}_stats.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
