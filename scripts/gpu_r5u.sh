# repair: fixed-offset record staging (no global atomic), first cells of 2 / 4 walks loaded together
mkdir -p gpurun_out
T=${TAG:-r5u}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_LIBRARY=ab/libmt_pre2fix.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
