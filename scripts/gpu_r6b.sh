# tile minima cells written as whole 32-B sectors by one 256-bit store (TILE_FULLSECTOR): time + DRAM bytes
mkdir -p gpurun_out
T=${TAG:-r6b}
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
for v in base fs; do MT_LIBRARY=ab/libmt_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tile_tmt|merge_queue|repair_brick" -s 3 -c 3 --csv python scripts/stats.py c5 > gpurun_out/${T}_dram_$v.csv 2>&1; done
MT_LIBRARY=ab/libmt_fs.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
