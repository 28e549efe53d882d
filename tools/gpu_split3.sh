timeout 900 python -m pytest tests/test_gpu_spec.py -x -q -k "split or matches_oracle" 2>&1 | tail -2
python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=4,spec:CUPSO_SPEC_CFG=5,spec:CUPSO_SPEC_CFG=6,spec:CUPSO_SPEC_CFG=7 6 2>&1
