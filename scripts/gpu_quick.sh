# quick GPU iteration: parity (small/medium, per-test timeout) + per-kernel times and counters
mkdir -p gpurun_out
T=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python scripts/stats.py ${CFGS:-c2 c3 c4 c5} > gpurun_out/${T}_stats.log 2>&1
if [ -n "$PROF" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${PROF}" -s ${SKIP:-3} -c 1 -o gpurun_out/${T}_prof python bench.py --config ${PCFG:-c5} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_prof.log 2>&1
fi
