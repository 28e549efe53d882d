python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=1,spec:CUPSO_SPEC_CFG=2,spec:CUPSO_SPEC_CFG=3,spec:CUPSO_SPEC_CFG=4 0,1 2>&1
python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=1,spec:CUPSO_SPEC_CFG=2 2,3 2>&1
