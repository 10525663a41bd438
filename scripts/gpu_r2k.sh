mkdir -p gpurun_out
T=r2k
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_graph.py -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
MT_LIBRARY=ab/libmt_nv8k.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest8k.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest8k.log
for c in c4 c5; do ROUNDS=9 timeout 600 python scripts/ab_interleave.py $c ab/libmt_both.so ab/libmt_none.so >> gpurun_out/${T}_ab.log 2>&1; done
