# merge_queue fetch batch and occupancy
mkdir -p gpurun_out
T=${TAG:-r5w}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
