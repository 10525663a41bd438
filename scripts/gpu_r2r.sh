mkdir -p gpurun_out
T=r2r
MT_LIBRARY=ab/libmt_new.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in c4 c5; do ROUNDS=9 timeout 600 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_atom_dot_cas.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
MT_LIBRARY=ab/libmt_new.so timeout 900 ncu --metrics $M --clock-control none -k regex:"merge_queue|forest" -s 1 -c 1 --csv --log-file gpurun_out/${T}_mq.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_mq.log 2>&1
MT_LIBRARY=ab/libmt_new.so timeout 900 python scripts/slab_estimate.py c5 8 > gpurun_out/${T}_slab.jsonl 2>&1
