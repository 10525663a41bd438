# f3 fixes (one-plane slabs, bounded O4 samples) + L2 prefetch A/B of the tile kernel
mkdir -p gpurun_out
T=${TAG:-r4b}
timeout 900 python -m pytest tests/test_gpu_dist.py -q --timeout 600 > gpurun_out/${T}_pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_dist.log
for c in c4 c5; do ROUNDS=7 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
MT_F3_BIG=1 timeout 2400 python -m pytest tests/test_gpu_f3_big.py -q -s --timeout 2400 > gpurun_out/${T}_f3_big.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_f3_big.log
