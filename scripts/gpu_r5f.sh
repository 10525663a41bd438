# tile Alg. 3 path splitting (TILE_CSPLIT), id-range repair bricks (timing), new merge_queue defaults
mkdir -p gpurun_out
T=${TAG:-r5f}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_tcs.so timeout 600 python scripts/stats.py c5 > gpurun_out/${T}_stats_tcs.jsonl 2>&1
MT_LIBRARY=ab/libmt_tcs.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest_tcs.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_tcs.log
