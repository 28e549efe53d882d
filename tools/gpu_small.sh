python tools/spec_perf.py spec,spec:CUPSO_SPEC_CFG=1,spec:CUPSO_SPEC_CFG=3,resident,persistent 7,8,10 2>&1
python tools/spec_perf.py auto 9 2>&1
QP_VARIANTS=QUEUE_LOCK,REDUCTION python - <<'PY'
import sys, os
sys.path.insert(0, '.')
import paper_2205_01313_b200 as cp
for fit, n, d, T in [("cubic", 2048, 1, 100000), ("cubic", 65536, 1, 10000)]:
    f = cp.find_fitness(fit); p = cp.make_params(f, n, d, T)
    for v in (cp.QUEUE_LOCK, cp.REDUCTION, cp.ASYNC, cp.SYNC_F32):
        with cp.Swarm(p, f, 1) as sw:
            s = sw.step(v, T)
            print(fit, n, d, T, cp.lib().cupso_variant_name(v).decode(), f"{s:.4f} s {n*T/s:.3e} p-u/s", flush=True)
PY
