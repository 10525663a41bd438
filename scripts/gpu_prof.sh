# ncu capture of one kernel: KREGEX, CFG, SKIP (launches to skip) -> gpurun_out/${TAG}_prof.ncu-rep
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-4} -c ${COUNT:-1} -o gpurun_out/${TAG}_prof python bench.py --config ${CFG:-c4} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_prof.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_prof.log
