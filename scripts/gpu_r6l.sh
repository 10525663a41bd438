# final default (diagram 2 segments per thread): parity tests + full c5 O1 memcmp + bench
mkdir -p gpurun_out
T=${TAG:-r6l}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
MT_FULL_C5=1 timeout 2400 python -m pytest tests/test_gpu_full_c5.py -q -s --timeout 2400 > gpurun_out/${T}_c5full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_c5full.log
