# round-1 measurement pass: smoke, bench, launch list, ncu full captures
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -3 gpurun_out/bench_default.err
cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2>&1; cat gpurun_out/bench_reference.json | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --iters 50 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; tail -2 gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sync -c 1 -o gpurun_out/prof_sync_cfg2 python bench.py --steps 1 --warmup 0 --iters 200 --no-cpu --no-baseline-kernel > gpurun_out/ncu_sync.log 2>&1; tail -3 gpurun_out/ncu_sync.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_classic -s 200 -c 2 -o gpurun_out/prof_reduction_cfg2 python bench.py --variant cuda-reduction --steps 1 --warmup 0 --iters 200 --no-cpu --no-baseline-kernel > gpurun_out/ncu_red.log 2>&1; tail -3 gpurun_out/ncu_red.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sync -c 1 -o gpurun_out/prof_sync_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 0 --iters 10 --no-cpu --no-baseline-kernel > gpurun_out/ncu_sync4.log 2>&1; tail -3 gpurun_out/ncu_sync4.log
ls -la gpurun_out
