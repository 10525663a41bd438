# full round: all GPU tests, the default bench line, ncu launch list + full capture of the top kernels
mkdir -p gpurun_out
T=${TAG:-R}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|dedupe_cross|merge_queue|repair_brick|diagram_kernel" -s 12 -c 4 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full.log 2>&1
