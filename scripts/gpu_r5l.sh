# per-line profile of tile_tmt (refilling insert ring) at c5
mkdir -p gpurun_out
T=${TAG:-r5l}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt" -s 2 -c 1 -o gpurun_out/${T}_tile python scripts/stats.py c5 > gpurun_out/${T}_tile.log 2>&1
