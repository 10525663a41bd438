# stepped crossing-edge queue (no global atomic per dedupe step) + fixed-offset repair staging; full GPU tests
mkdir -p gpurun_out
T=${TAG:-r5v}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in c5 c4; do ROUNDS=7 timeout 900 python scripts/ab_interleave.py $c ab/libmt_*.so >> gpurun_out/${T}_ab.log 2>&1; done
