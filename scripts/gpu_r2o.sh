mkdir -p gpurun_out
T=r2o
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q --timeout 300 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
MT_BIG_IDS=1 timeout 1800 python -m pytest tests/test_gpu_big_ids.py -q -s --timeout 1800 > gpurun_out/${T}_bigids.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bigids.log
