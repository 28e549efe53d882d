timeout 900 python -m pytest tests/test_gpu_f32.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in cfg2 cfg3 cfg5; do timeout 900 python bench.py --workload $w --variant cuda-sync-f32 --no-cpu --steps 5 > gpurun_out/bench_f32_$w.json 2> gpurun_out/bench_f32_$w.err; tail -1 gpurun_out/bench_f32_$w.err; done
