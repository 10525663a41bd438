mkdir -p gpurun_out
T=r3f
MT_LIBRARY=ab/libmt_new.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in c4 c5; do ROUNDS=9 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_new.so timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
