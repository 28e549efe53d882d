for m in wave persistent; do CUPSO_SYNC_MODE=$m timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches and sync or final_state or golden or acceptance_per_iteration" 2>&1 | tail -1; done
for m in wave persistent; do echo "=== $m"; CUPSO_SYNC_MODE=$m CUPSO_STEP_CFG=0 QP_VARIANTS=SYNC timeout 300 python tools/quick_perf.py 4 2>&1 | grep cuda; done
QP_VARIANTS=QUEUE_LOCK timeout 300 python tools/quick_perf.py 4 2>&1 | grep cuda
