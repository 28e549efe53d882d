CUPSO_ASYNC_MODE=reg python tools/areg_diag.py cubic 20 1 200
CUPSO_ASYNC_MODE=reg timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_async_reg -c 1 -o gpurun_out/areg_c20 python tools/areg_diag.py cubic 20 1 64 > /dev/null 2>&1
CUPSO_SYNC_MODE=spec timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 6 -c 1 -o gpurun_out/spec_c20 python tools/prof_case.py cuda-sync cubic 20 1 200 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/areg_c20.ncu-rep gpurun_out/spec_c20.ncu-rep > gpurun_out/areg_ncu.txt 2>&1
