# merge_queue: no filter walks (MQ_WALK 0), path splitting inside the Alg. 3 climbs (MQ_CSPLIT), occupancy
mkdir -p gpurun_out
T=${TAG:-r5e}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
for v in w0csb4 w0b4; do MT_LIBRARY=ab/libmt_$v.so timeout 600 python scripts/stats.py c5 > gpurun_out/${T}_stats_$v.jsonl 2>&1; done
MT_LIBRARY=ab/libmt_w0csb4.so timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "parity or full_size or dist" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
