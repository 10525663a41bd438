# diagram kernel: segments per thread on big grids (DG_SPT_BIG 2 / 4 / 8)
mkdir -p gpurun_out
T=${TAG:-r6k}
for c in c5 c4; do ROUNDS=9 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_dg8.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "full_size or c5" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
