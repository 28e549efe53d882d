"""Quick device-time probe of every variant on a few shapes (exploration only)."""
import sys, time
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2205_01313_b200 as cp

VARIANTS = [getattr(cp, v) for v in __import__("os").environ.get("QP_VARIANTS", "SYNC,ASYNC,QUEUE_LOCK,QUEUE,REDUCTION").split(",")]
shapes = [("cubic", 1 << 20, 1, 200), ("cubic", 1 << 24, 1, 20), ("rastrigin", 1 << 20, 32, 10), ("sphere", 1 << 24, 8, 10)]
if len(sys.argv) > 1:
    shapes = shapes[: int(sys.argv[1])]
for fit, n, d, T in shapes:
    f = cp.find_fitness(fit)
    p = cp.make_params(f, n, d, T)
    with cp.Swarm(p, f, 1) as sw:
        for v in VARIANTS:
            best = 1e9
            for rep in range(2):
                sw.init()
                s = sw.step(v, T)
                best = min(best, s)
            pus = n * T / best
            gbs = pus * (5 * d + 1) * 8 / 1e9
            print(f"{fit:10s} n=2^{n.bit_length()-1} d={d:3d} T={T:4d} {cp.lib().cupso_variant_name(v).decode():16s} "
                  f"{best*1e6/T:9.2f} us/iter  {pus:.3e} p-u/s  {gbs:8.1f} GB/s  grid={sw.sync_grid_blocks()}  gbest={sw.gbest().fit:.6g}", flush=True)
