for D in 0 1 2 4 7; do CUPSO_AREG_DIAG=$D CUPSO_ASYNC_MODE=reg python tools/areg_diag.py cubic 20 1 200 | sed "s/^/diag=$D /"; done
