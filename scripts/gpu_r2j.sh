mkdir -p gpurun_out
T=r2j
for c in c3 c4 c5; do ROUNDS=7 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
