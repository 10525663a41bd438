mkdir -p gpurun_out
timeout 120 python scripts/dist_debug.py c4 32 2 > gpurun_out/${TAG}_debug.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_debug.log
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -x -q --timeout 120 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
