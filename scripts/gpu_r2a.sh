# round 2, call a: GPU tests, per-phase stats, bench, then the full-size c5 O1 memcmp
mkdir -p gpurun_out
T=${TAG:-r2a}
nproc > gpurun_out/${T}_host.txt; free -g >> gpurun_out/${T}_host.txt; lscpu | head -20 >> gpurun_out/${T}_host.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python scripts/stats.py c3 c4 c5 > gpurun_out/${T}_stats.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
MT_FULL_C5=1 timeout 2400 python -m pytest tests/test_gpu_full_c5.py -q -s --timeout 2400 > gpurun_out/${T}_c5full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_c5full.log
