mkdir -p gpurun_out
T=r2f
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for lib in ab/libmt_*.so; do
  echo "== $lib" >> gpurun_out/${T}_ab.log
  MT_LIBRARY=$lib timeout 300 python scripts/stats.py c4 c5 >> gpurun_out/${T}_ab.log 2>&1
done
