timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "async" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "async" 2>&1 | tail -2
for K in 8 32 64; do CUPSO_ASYNC_K=$K CUPSO_ASYNC_MODE=reg python tools/areg_diag.py cubic 20 1 200; done
CUPSO_ASYNC_MODE=reg python tools/areg_diag.py cubic 24 1 100
CUPSO_ASYNC_MODE=tiled python tools/areg_diag.py cubic 24 1 100
CUPSO_ASYNC_MODE=reg python tools/areg_diag.py sphere 20 8 100
CUPSO_ASYNC_MODE=reg python tools/areg_diag.py sphere 24 8 50
