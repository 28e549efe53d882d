python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
bash tools/gpu_ncu.sh r01_cfg2_sync k_sync_res 0 cuda-sync cubic 20 1 200
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -2 gpurun_out/bench_cfg2.err
