# final-code verification: every GPU test, smoke, the f3 4.33e9-vertex slab test, the ids >= 2^31 test, bench c5
mkdir -p gpurun_out
T=${TAG:-r6j}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
MT_F3_BIG=1 timeout 2400 python -m pytest tests/test_gpu_f3_big.py -q -s --timeout 2400 > gpurun_out/${T}_f3_big.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_f3_big.log
MT_BIG_IDS=1 timeout 2400 python -m pytest tests/test_gpu_big_ids.py -q -s --timeout 2400 > gpurun_out/${T}_big_ids.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_big_ids.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
MT_DIST_BACKEND=gloo MT_FORCE_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config c4 --no-e2e > gpurun_out/${T}_multi2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_multi2_gloo.log
