# minima normalisation pass: GPU tests, stats (hop counts), interleaved A/B against the build without it
mkdir -p gpurun_out
T=${TAG:-r5b}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python scripts/stats.py c4 c5 > gpurun_out/${T}_stats.jsonl 2>&1
MT_LIBRARY=ab/libmt_nonorm.so timeout 600 python scripts/stats.py c5 > gpurun_out/${T}_stats_nonorm.jsonl 2>&1
for c in c4 c5; do ROUNDS=7 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
