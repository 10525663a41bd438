# A/B: per-kernel times of each variant library under ab/ (scripts/ab_build.py) on ${CFGS:-c5};
# EXTRA="ENV=VAL lib" adds one run of ab/libmt_<lib>.so under an environment override
mkdir -p gpurun_out
T=${TAG:-ab}
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 -k "not full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log; fi
for lib in ab/libmt_*.so; do
  echo "== $lib" >> gpurun_out/${T}_ab.log
  MT_LIBRARY=$lib timeout 300 python scripts/stats.py ${CFGS:-c5} >> gpurun_out/${T}_ab.log 2>&1
done
if [ -n "$EXTRA" ]; then
  set -- $EXTRA
  echo "== $1:$2" >> gpurun_out/${T}_ab.log
  env $1 MT_LIBRARY=ab/libmt_$2.so timeout 300 python scripts/stats.py ${CFGS:-c5} >> gpurun_out/${T}_ab.log 2>&1
fi
