mkdir -p gpurun_out
T=${TAG:-m}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/${T}_san_${tool}.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_san_${tool}.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>&1; echo "rc=$?" >> gpurun_out/${T}_ref.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|merge_queue|repair_brick|diagram_kernel|dedupe_cross" -s 12 -c 4 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_full.log 2>&1
