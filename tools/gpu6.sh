set -x
CUPSO_STEP_CFG=5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sync -c 1 -o gpurun_out/prof_sync5_sphere python tools/prof_case.py cuda-sync sphere 24 8 3 > gpurun_out/p1.log 2>&1; tail -2 gpurun_out/p1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_classic_step -s 2 -c 1 -o gpurun_out/prof_ql_sphere python tools/prof_case.py cuda-queue-lock sphere 24 8 4 > gpurun_out/p2.log 2>&1; tail -2 gpurun_out/p2.log
