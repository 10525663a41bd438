# one GPU round: parity tests, diagnostics, benches, ncu of the merge kernel
mkdir -p gpurun_out
T=${TAG:-r}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "full_size" > gpurun_out/${T}_pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_full.log
timeout 600 python scripts/stats.py c2 c3 c4 c5 > gpurun_out/${T}_stats.log 2>&1
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_c4.log 2>&1
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/${T}_bench_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_cross -s 3 -c 1 -o gpurun_out/${T}_merge_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|repair_brick|diagram_kernel" -s 6 -c 2 -o gpurun_out/${T}_other_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_*.log
