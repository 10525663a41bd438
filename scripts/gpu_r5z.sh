# bench sanity on the final build: default line (e2e over 10 steps) and the reference arm
mkdir -p gpurun_out
T=${TAG:-r5z}
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>&1; echo "rc=$?" >> gpurun_out/${T}_ref.json
