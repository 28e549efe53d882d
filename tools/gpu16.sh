timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for w in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_cfg2.json 2>&1
