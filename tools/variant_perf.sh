# compare library variants on cfg2/cfg4/cfg5-proxy (device time only)
for v in build/variants/*.so; do
  echo "=== $v"
  CUPSO_LIB=$PWD/$v timeout 300 python tools/quick_perf.py 4 2>&1 | grep -E "cuda-sync|cuda-async|cuda-reduction|queue-lock"
done
