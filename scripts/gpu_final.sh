# round checkpoint: all GPU tests, bench lines (c5 default, c4), ncu launch list + full capture,
# sanitizers on small configs, the reference (oracle) arm
mkdir -p gpurun_out
T=${TAG:-F}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 15 -c 5 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/${T}_san_${tool}.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_san_${tool}.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>&1; echo "rc=$?" >> gpurun_out/${T}_ref.json
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2>&1
MT_DIST_BACKEND=gloo MT_FORCE_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config c4 --no-e2e > gpurun_out/${T}_multi2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_multi2_gloo.log
