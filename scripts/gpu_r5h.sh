# repair walks chained in threshold order (MT_REPAIR_CHAIN) vs base
mkdir -p gpurun_out
T=${TAG:-r5h}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_chain.so timeout 600 python scripts/stats.py c5 > gpurun_out/${T}_stats_chain.jsonl 2>&1
MT_LIBRARY=ab/libmt_chain.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_graph.py -x -q --timeout 600 > gpurun_out/${T}_pytest_chain.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_chain.log
