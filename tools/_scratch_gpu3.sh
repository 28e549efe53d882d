python -m pytest tests/test_gpu_stats.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -q -x -s 2>&1 | grep -v "^$" | tail -12
python -m pytest tests/test_gpu_scale.py -q -x -k "async" 2>&1 | tail -3
python bench.py --workload cfg3 --steps 3 --no-cpu --no-baseline-kernel --no-strong --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['roofline'].get('mode'))"
python bench.py > gpurun_out/bench_cfg2_r02b.json 2> gpurun_out/bench_cfg2_r02b.err; tail -c 600 gpurun_out/bench_cfg2_r02b.err
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2_r02b.json').read().splitlines()[-1]); print(json.dumps({k: d[k] for k in ('value','e2e','strong_cfg5','paper_engines','reduction_baseline','gpu_launches')}, indent=0)); print(json.dumps(d['roofline'])[:1500])"
timeout 900 python tools/ncu_bench.py r02 cfg2 cfg4 2>&1 | tail -5
