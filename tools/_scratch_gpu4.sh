python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 1500 python tools/ncu_bench.py r02 cfg3 cfg5 2>&1 | tail -3
python bench.py --no-strong --no-cpu > gpurun_out/bench_cfg2_r02c.json 2> gpurun_out/bench_cfg2_r02c.err; python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2_r02c.json').read().splitlines()[-1]); r=d['roofline']; print(d['value'], d['gpu_launches'], r['bound'], r['frac'], r.get('traffic'), r['spec'])"
