set -x
for c in 0 2 5; do CUPSO_STEP_CFG=$c timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches and sync or final_state or golden" 2>&1 | tail -2; done
bash tools/cfg_sweep.sh
QP_VARIANTS=QUEUE_LOCK,QUEUE,REDUCTION,UNROLLED timeout 300 python tools/quick_perf.py 4
