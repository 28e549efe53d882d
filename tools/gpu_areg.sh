timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "async" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "async" 2>&1 | tail -3
for m in reg tiled plain; do CUPSO_ASYNC_MODE=$m QP_VARIANTS=ASYNC python tools/quick_perf.py 2 2>&1 | sed "s/^/$m /"; done
