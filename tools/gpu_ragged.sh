timeout 1200 python -m pytest tests/test_gpu_spec.py tests/test_gpu_scale.py -x -q 2>&1 | tail -3
python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=8,spec:CUPSO_SPEC_CFG=7 6 2>&1
python tools/spec_perf.py spec,wave 8,9,10 2>&1
