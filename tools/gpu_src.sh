# source-level (SASS) stall sampling of one k_spec pass (cfg2 shape); only CSVs travel back
export CUPSO_SYNC_MODE=spec
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spec -s 8 -c 1 -o /tmp/src_c2 python tools/prof_case.py cuda-sync cubic 20 1 600 > /dev/null 2>&1
ncu -i /tmp/src_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/src_c2.csv 2>/dev/null
ncu -i /tmp/src_c2.ncu-rep --page raw --csv > gpurun_out/raw_c2.csv 2>/dev/null
ls -la gpurun_out/src_c2.csv gpurun_out/raw_c2.csv
