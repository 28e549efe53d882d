timeout 900 python -m pytest tests/test_gpu_spec.py -x -q 2>&1 | tail -3
python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=5,spec:CUPSO_SPEC_CFG=6 0,1 2>&1
python tools/spec_perf.py spec,wave 2,3,4,5 2>&1
