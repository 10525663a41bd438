# tile: refilling hash insert (TILE_RINS), warp-shared in-tile repair walks (TILE_RREP); diagram prefetch; dedupe 32-bit minima
mkdir -p gpurun_out
T=${TAG:-r5k}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_both.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest_both.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_both.log
MT_LIBRARY=ab/libmt_dcm32.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest_dcm32.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_dcm32.log
