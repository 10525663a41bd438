mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r1_info.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "not full_size" > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "full_size" > gpurun_out/r1_pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/r1_pytest_full.log
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/r1_bench_c4.log 2>&1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_c3.log 2>&1
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_c2.log 2>&1
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r1_bench_c5.log 2>&1
tail -3 gpurun_out/*.log
