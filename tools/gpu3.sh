set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches or final_state or golden" 2>&1 | tail -4
bash tools/variant_perf.sh
