for c in 2 5 6 7; do echo "=== cfg $c"; CUPSO_STEP_CFG=$c QP_VARIANTS=SYNC timeout 300 python tools/quick_perf.py 4 2>&1 | grep cuda; done
