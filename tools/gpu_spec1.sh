# spec mode: parity suite, then the whole GPU suite, then mode timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py -x -q 2>&1 | tail -15
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 900 python tools/spec_perf.py spec,resident,wave 2>&1 | tee gpurun_out/spec_perf1.txt
