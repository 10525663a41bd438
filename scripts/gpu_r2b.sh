# round 2, call b: N11 microbenchmarks, dist/graph/c5-sampled tests, tile_tmt source-level ncu, atomic counters per kernel
mkdir -p gpurun_out
T=${TAG:-r2b}
timeout 300 python scripts/n11.py > gpurun_out/${T}_n11.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_graph.py "tests/test_gpu_parity.py::test_full_size_c5_sampled" -q --timeout 600 -s > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_requests_op_atom.sum,lts__t_requests_op_atom_dot_cas.sum,lts__t_sectors_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,sm__sass_inst_executed_op_global_atom.sum,sm__sass_inst_executed_op_shared_atom.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 900 ncu --metrics $M --clock-control none -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 10 -c 5 --csv --log-file gpurun_out/${T}_atom.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_atom.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tile_tmt -s 3 -c 1 -o gpurun_out/${T}_tile python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_tile.log 2>&1
