"""Where the e2e time of cupso_run goes (exploration): wall time of find_engine(...).run
vs its device compute_seconds, at T = 1000 and T = 1 (fixed per-call overhead)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01313_b200 as cp
f = cp.find_fitness("cubic")
for T in (1000, 1):
    p = cp.make_params(f, 1 << 20, 1, T)
    e = cp.find_engine("cuda-sync")
    e.run(p, f, cp.rng_key(1))
    walls, devs = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        r = e.run(p, f, cp.rng_key(1))
        walls.append(time.perf_counter() - t0)
        devs.append(r.compute_seconds)
    w, d = sum(walls) / len(walls), sum(devs) / len(devs)
    print(f"T={T}: wall {w * 1e3:.3f} ms, device loop {d * 1e3:.3f} ms, overhead {(w - d) * 1e6:.0f} us")
