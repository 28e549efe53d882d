# ncu captures of the spec kernel (cfg2 shape, cfg5 proxy)
export CUPSO_SYNC_MODE=spec
bash tools/gpu_ncu.sh r01_spec_cfg2 k_spec 8 cuda-sync cubic 20 1 600
bash tools/gpu_ncu.sh r01_spec_cfg5p k_spec 12 cuda-sync sphere 24 8 50
python tools/ncu_summary.py gpurun_out/r01_spec_cfg2.ncu-rep gpurun_out/r01_spec_cfg5p.ncu-rep > gpurun_out/spec_ncu.txt 2>&1
ncu -i gpurun_out/r01_spec_cfg2.ncu-rep --page details --csv > gpurun_out/spec_cfg2_details.csv 2>&1
ncu -i gpurun_out/r01_spec_cfg5p.ncu-rep --page details --csv > gpurun_out/spec_cfg5p_details.csv 2>&1
