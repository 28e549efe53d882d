for c in 0 1 2 3 4; do
  echo "=== wave cfg $c"
  CUPSO_WAVE_CFG=$c timeout 300 python tools/prof_case.py cuda-sync sphere 24 8 10
  CUPSO_WAVE_CFG=$c timeout 300 python tools/prof_case.py cuda-sync rastrigin 20 32 10
  CUPSO_WAVE_CFG=$c timeout 300 python tools/prof_case.py cuda-sync sphere 22 64 5
done
CUPSO_WAVE_CFG=3 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "engine_matches and sync or modes or cfg5 or cfg4" 2>&1 | tail -2
