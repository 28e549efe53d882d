for K in 1 8 32; do CUPSO_ASYNC_MODE=reg CUPSO_ASYNC_K=$K python tools/areg_diag.py cubic 20 1 200; done
CUPSO_ASYNC_MODE=tiled python tools/areg_diag.py cubic 20 1 200
CUPSO_ASYNC_MODE=reg python tools/areg_diag.py sphere 20 8 100
CUPSO_ASYNC_MODE=tiled python tools/areg_diag.py sphere 20 8 100
