mkdir -p gpurun_out
for m in 4096 2048; do
  MT_TILE_NV=$m timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 -k "not full_size" > gpurun_out/${TAG}_m${m}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_m${m}_pytest.log
  MT_TILE_NV=$m timeout 600 python scripts/stats.py ${CFGS:-c2 c4 c5} > gpurun_out/${TAG}_m${m}_stats.log 2>&1
done
