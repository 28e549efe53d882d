set -x
for c in 2 5; do CUPSO_STEP_CFG=$c timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches and sync or final_state or golden" 2>&1 | tail -1; done
for c in 0 2 4 5; do echo "=== cfg $c"; CUPSO_STEP_CFG=$c QP_VARIANTS=SYNC,ASYNC timeout 300 python tools/quick_perf.py 4 2>&1 | grep cuda; done
CUPSO_STEP_CFG=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sync -c 1 -o gpurun_out/prof_sync2_sphere python tools/prof_case.py cuda-sync sphere 24 8 3 > gpurun_out/p1.log 2>&1; tail -1 gpurun_out/p1.log
