# round-1 measurement pass, part 1: bench lines (small outputs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_adapter.py -q -m gpu -s 2>&1 | tail -8
for w in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_cfg2.json 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
