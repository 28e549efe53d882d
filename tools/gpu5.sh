set -x
CUPSO_STEP_CFG=5 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches and sync or final_state or golden" 2>&1 | tail -2
bash tools/cfg_sweep.sh
