# tile: root keys from the cell in the merge loop (TILE_ROOTKEY), compaction unroll (TILE_CUNROLL)
mkdir -p gpurun_out
T=${TAG:-r6d}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_rk.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
