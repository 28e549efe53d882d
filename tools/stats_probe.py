"""Exploration: final-fitness distributions over 32 seeds of the statistical
engines (cuda-async, cuda-sync-f32) against run_serial's (cuda-sync, bitwise
run_serial) on non-degenerate fitnesses, with a Mann-Whitney U test.

    python tools/stats_probe.py [n] [T]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
from scipy.stats import mannwhitneyu  # noqa: E402

import paper_2205_01313_b200 as cp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = int(sys.argv[2]) if len(sys.argv) > 2 else 300
ENGINES = os.environ.get("PROBE_ENGINES", "cuda-async,cuda-sync-f32").split(",")
FITS = [(a.split(":")[0], int(a.split(":")[1])) for a in
        os.environ.get("PROBE_FITS", "sphere:8,rastrigin:32,griewank:8").split(",")]
for fit, d in FITS:
    f = cp.find_fitness(fit)
    p = cp.make_params(f, n, d, T)
    cost = {}
    for e in ["cuda-sync"] + ENGINES:
        cost[e] = np.array([-cp.find_engine(e).run(p, f, cp.rng_key(s)).gbest_fit for s in range(1, 33)])
    base = cost["cuda-sync"]
    print(f"{fit} d={d} n={n} T={T}: sync median {np.median(base):.6g} "
          f"q25/q75 {np.percentile(base, 25):.4g}/{np.percentile(base, 75):.4g}")
    for e in ENGINES:
        c = cost[e]
        u = mannwhitneyu(c, base, alternative="two-sided")
        print(f"   {e:14s} median {np.median(c):.6g} ratio {np.median(c) / max(np.median(base), 1e-300):.3f} "
              f"q25/q75 {np.percentile(c, 25):.4g}/{np.percentile(c, 75):.4g}  MWU p={u.pvalue:.4f}")
