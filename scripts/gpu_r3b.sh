mkdir -p gpurun_out
T=r3b
MT_LIBRARY=ab/libmt_r32m4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_graph.py -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in c4 c5; do ROUNDS=9 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
