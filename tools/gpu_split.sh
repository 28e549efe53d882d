timeout 900 python -m pytest tests/test_gpu_spec.py -x -q 2>&1 | tail -3
python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=1,spec:CUPSO_SPEC_CFG=2,spec:CUPSO_SPEC_CFG=3,wave 6 2>&1
