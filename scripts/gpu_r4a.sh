# f3 wide ids: all GPU tests (incl. the wide-mode virtual-rank parity), the 2-rank gloo bench,
# the slab estimate, then the 4.33e9-vertex grid in 8 slabs
mkdir -p gpurun_out
T=${TAG:-r4a}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
MT_DIST_BACKEND=gloo MT_FORCE_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config c4 --no-e2e > gpurun_out/${T}_multi2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_multi2_gloo.log
timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
MT_F3_BIG=1 timeout 2400 python -m pytest tests/test_gpu_f3_big.py -q -s --timeout 2400 > gpurun_out/${T}_f3_big.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_f3_big.log
