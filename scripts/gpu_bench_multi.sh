mkdir -p gpurun_out
# multi-rank path on one GPU: ranks share cuda:0 over gloo (NCCL refuses two ranks per GPU)
for N in ${NS:-2}; do
MT_DIST_BACKEND=gloo MT_FORCE_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 3 --warmup 3 --config ${CFG:-c4} > gpurun_out/${TAG}_multi${N}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_multi${N}.log
done
