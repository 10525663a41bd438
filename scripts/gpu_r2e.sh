mkdir -p gpurun_out
T=r2e
for lib in ab/libmt_*.so; do
  echo "== $lib" >> gpurun_out/${T}_ab.log
  MT_LIBRARY=$lib timeout 300 python scripts/stats.py c5 >> gpurun_out/${T}_ab.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"repair_brick|tile_tmt" -s 6 -c 2 -o gpurun_out/${T}_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_prof.log 2>&1
