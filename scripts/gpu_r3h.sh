mkdir -p gpurun_out
T=r3h
MT_LIBRARY=ab/libmt_nv8k.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --timeout 300 -k "not full_size and not launches" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in c4 c5; do ROUNDS=7 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
