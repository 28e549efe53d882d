set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_spec.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -8
python tools/quick_shape.py rastrigin 1048576 32 1000
python tools/quick_shape.py griewank 1048576 8 300
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg4', d['value'], d['reduction_baseline'])"
for K in 1 4 8 16; do CUPSO_ASYNC_K=$K PROBE_ENGINES=cuda-async PROBE_FITS=sphere:8,griewank:8 python tools/stats_probe.py 4096 300 | sed "s/^/K=$K /"; done
PROBE_ENGINES=cuda-async PROBE_FITS=sphere:8,griewank:8 python tools/stats_probe.py 65536 300 | sed "s/^/n=65536 /"
