# round-2 session 3, first call: smoke, stats (counters + per-kernel times) c4/c5, and ncu --set full with
# source of tile_tmt and repair_brick at c5 (for per-line instruction / stall attribution)
mkdir -p gpurun_out
T=${TAG:-r5a}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python scripts/stats.py c4 c5 > gpurun_out/${T}_stats.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile_tmt|repair_brick" -s 4 -c 2 -o gpurun_out/${T}_full python scripts/stats.py c5 > gpurun_out/${T}_full.log 2>&1
