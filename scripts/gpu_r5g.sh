# forest_merge with climb splitting (FM_CSPLIT): dist parity tests + virtual-rank estimate vs FM_CSPLIT=0
mkdir -p gpurun_out
T=${TAG:-r5g}
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_graph.py -x -q --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python scripts/slab_estimate.py c5 2 4 8 > gpurun_out/${T}_slab.jsonl 2>&1
MT_LIBRARY=ab/libmt_fm0.so timeout 900 python scripts/slab_estimate.py c5 8 > gpurun_out/${T}_slab_fm0.jsonl 2>&1
