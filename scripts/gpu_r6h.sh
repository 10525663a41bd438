# forest face records at fixed slots, boundary dedupe without id lookups (FOREST_FACEIDX): dist parity + P estimate
mkdir -p gpurun_out
T=${TAG:-r6h}
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q --timeout 600 > gpurun_out/${T}_pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_dist.log
timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
MT_LIBRARY=ab/libmt_nofi.so timeout 900 python scripts/slab_estimate.py c5 8 > gpurun_out/${T}_slab_nofi.jsonl 2>&1
