# tile merge stragglers parked and finished packed (TILE_TAIL); repair chain with the stopping cell kept (MT_REPAIR_CHAIN)
mkdir -p gpurun_out
T=${TAG:-r5t}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_tail6.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest_tail.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_tail.log
MT_LIBRARY=ab/libmt_chain.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --timeout 600 > gpurun_out/${T}_pytest_chain.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_chain.log
