mkdir -p gpurun_out
T=${TAG:-b}
timeout 900 python bench.py ${ARGS} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
