# repair brick order: the two bricks of a tile depth back to back (ZPAIR), tile-deep bricks (ROWS 128)
mkdir -p gpurun_out
T=${TAG:-r5i}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_zp.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest_zp.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_zp.log
MT_LIBRARY=ab/libmt_r128.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/${T}_pytest_r128.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_r128.log
