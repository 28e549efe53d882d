# bench lines for every workload (+ reference arm) -> gpurun_out/bench_*.json
mkdir -p gpurun_out
for w in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err
done
