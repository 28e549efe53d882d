"""Diagnose async register mode: occupancy per iteration, timing vs K."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_01313_b200 as cp
fit, lg, d, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
f = cp.find_fitness(fit)
p = cp.make_params(f, 1 << lg, d, 2 * T)
with cp.Swarm(p, f, 1) as sw:
    s = sw.step(cp.ASYNC, T)
    s2 = sw.step(cp.ASYNC, T)
    print(f"steady-state (second {T} iterations): {s2*1e6/T:.2f} us/iter")
    tr, tp, oc = sw.trace()
    print(f"{os.environ.get('CUPSO_ASYNC_MODE')} K={os.environ.get('CUPSO_ASYNC_K')} {s*1e6/T:.2f} us/iter; "
          f"occupancy first 5 {oc[:5]} sum {oc.sum():.4g}; trace changes {np.count_nonzero(np.diff(tr))}; final {tr[-1]}")
