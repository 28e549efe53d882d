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

# pieces through the handle API (each call synchronises)
import numpy as np
p = cp.make_params(f, 1 << 20, 1, 1000)
with cp.Swarm(p, f, 1) as sw:
    ts = {"init": [], "step1": [], "gbest": [], "trace": []}
    for _ in range(10):
        t0 = time.perf_counter(); sw.init(); t1 = time.perf_counter()
        sw.step(cp.SYNC, 1); t2 = time.perf_counter()
        sw.gbest(); t3 = time.perf_counter()
        sw.trace(0, 1); t4 = time.perf_counter()
        for k, a, b in (("init", t0, t1), ("step1", t1, t2), ("gbest", t2, t3), ("trace", t3, t4)):
            ts[k].append(b - a)
    print("handle API, us per call:", {k: round(1e6 * float(np.median(v)), 1) for k, v in ts.items()})
# the raw C call without the Python result wrapper
from paper_2205_01313_b200 import _lib
p1 = cp.make_params(f, 1 << 20, 1, 1)
cpar = p1.to_c()
g = np.zeros(1); tr = np.zeros(1); tp = np.zeros(1, np.uint32); oc = np.zeros(1)
import ctypes as C
res = _lib.cupso_result(0.0, 0, 0.0, 0.0, g.ctypes.data_as(C.POINTER(C.c_double)), tr.ctypes.data_as(C.POINTER(C.c_double)),
                        tp.ctypes.data_as(C.POINTER(C.c_uint32)), oc.ctypes.data_as(C.POINTER(C.c_double)), 0)
fn = _lib.OBSERVER_FN()
w = []
for _ in range(20):
    t0 = time.perf_counter()
    cp.lib().cupso_run(C.byref(cpar), f.id, 1, cp.SYNC, 0, fn, None, C.byref(res))
    w.append(time.perf_counter() - t0)
print(f"raw cupso_run T=1: {1e6 * float(np.median(w[2:])):.1f} us")
