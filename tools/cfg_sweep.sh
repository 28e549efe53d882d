# sweep the fused-step tunings (CUPSO_STEP_CFG) on the four workload shapes
for c in 0 1 2 3 4 5; do
  echo "=== cfg $c"
  CUPSO_STEP_CFG=$c QP_VARIANTS=SYNC,ASYNC timeout 300 python tools/quick_perf.py 4 2>&1 | grep -E "cuda-sync|cuda-async"
done
