# dedupe_cross patch rows 8 (256-thread steps) vs 16
mkdir -p gpurun_out
T=${TAG:-r6n}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
