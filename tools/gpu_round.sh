# full check: smoke, GPU suite, bench lines for every workload (+ FP32 engine), reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for w in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err
done
for w in cfg2 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --variant cuda-sync-f32 --no-cpu > gpurun_out/bench_f32_$w.json 2> gpurun_out/bench_f32_$w.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_cfg2.json 2>&1
