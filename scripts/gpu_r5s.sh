# repair timing stops: T0 -> T stream alone (1), + minima cells and records (2), vs the full repair
mkdir -p gpurun_out
T=${TAG:-r5s}
for c in c5; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
