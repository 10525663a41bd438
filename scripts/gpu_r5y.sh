# round-2 session-3 checkpoint: all GPU tests, smoke, bench lines (c5 default + c4, c3, c2 with more steps), ncu launch list
# + full capture of all six kernels, per-kernel atomics, reference arm, 2-rank gloo bench, full c5 O1 memcmp
mkdir -p gpurun_out
T=${TAG:-r5y}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2>&1
for c in c3 c2; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 18 -c 6 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_atom_dot_cas.sum,sm__sass_inst_executed_op_shared_atom.sum,sm__sass_inst_executed_op_global_atom.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct
timeout 900 ncu --metrics $M --clock-control none -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 18 -c 6 --csv --log-file gpurun_out/${T}_atom.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_atom.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>&1; echo "rc=$?" >> gpurun_out/${T}_ref.json
MT_DIST_BACKEND=gloo MT_FORCE_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --config c4 --no-e2e > gpurun_out/${T}_multi2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_multi2_gloo.log
timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
MT_FULL_C5=1 timeout 2400 python -m pytest tests/test_gpu_full_c5.py -q -s --timeout 2400 > gpurun_out/${T}_c5full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_c5full.log
MT_BIG_IDS=1 timeout 2400 python -m pytest tests/test_gpu_big_ids.py -q -s --timeout 2400 > gpurun_out/${T}_big_ids.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_big_ids.log
MT_F3_BIG=1 timeout 2400 python -m pytest tests/test_gpu_f3_big.py -q -s --timeout 2400 > gpurun_out/${T}_f3_big.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_f3_big.log
