# tile_tmt A/B: hash insert with one CAS site (TILE_INS2), merge refill threshold (TILE_REFILL), origin by thread 0
mkdir -p gpurun_out
T=${TAG:-r5c}
for c in c4 c5; do ROUNDS=9 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
