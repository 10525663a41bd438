# round-2 checkpoint: all GPU tests, smoke, bench lines, ncu launch list + full capture, full c5 O1 memcmp, reference arm
mkdir -p gpurun_out
T=${TAG:-r2q}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
for c in c4 c3 c2; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 15 -c 5 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_atom_dot_cas.sum,sm__sass_inst_executed_op_shared_atom.sum,sm__sass_inst_executed_op_global_atom.sum,smsp__inst_executed.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct
timeout 900 ncu --metrics $M --clock-control none -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 15 -c 5 --csv --log-file gpurun_out/${T}_atom.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_atom.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>&1; echo "rc=$?" >> gpurun_out/${T}_ref.json
MT_FULL_C5=1 timeout 2400 python -m pytest tests/test_gpu_full_c5.py -q -s --timeout 2400 > gpurun_out/${T}_c5full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_c5full.log
