# face-aware forest lookups (face records found by position, not in the id table): dist parity, f3 big, estimate
mkdir -p gpurun_out
T=${TAG:-r6i}
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q --timeout 600 > gpurun_out/${T}_pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_dist.log
timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
MT_LIBRARY=ab/libmt_nofi.so timeout 900 python scripts/slab_estimate.py c5 8 > gpurun_out/${T}_slab_nofi.jsonl 2>&1
MT_F3_BIG=1 timeout 2400 python -m pytest tests/test_gpu_f3_big.py -q -s --timeout 2400 > gpurun_out/${T}_f3_big.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_f3_big.log
