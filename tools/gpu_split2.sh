export CUPSO_SYNC_MODE=spec
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 6 -c 1 -o gpurun_out/split_c4 python tools/prof_case.py cuda-sync rastrigin 20 32 100 > gpurun_out/split_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/split_c4.ncu-rep > gpurun_out/split_ncu.txt 2>&1
