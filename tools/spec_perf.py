"""Device time of cuda-sync's modes on the BASELINE shapes (exploration; CUPSO_SYNC_MODE per process)."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CODE = r'''
import sys, json; sys.path.insert(0, %r)
import paper_2205_01313_b200 as cp
fit, n, d, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
f = cp.find_fitness(fit); p = cp.make_params(f, n, d, T)
with cp.Swarm(p, f, 1) as sw:
    best = 1e9
    for rep in range(3):
        sw.init(); best = min(best, sw.step(cp.SYNC, T))
    print(json.dumps(dict(mode=sw.sync_mode(), us_iter=best * 1e6 / T, pus=n * T / best,
                          gbs=n * T / best * (5 * d + 1) * 8 / 1e9, stats=sw.spec_stats(), gbest=sw.gbest().fit)))
''' % ROOT
shapes = [("cubic", 1 << 20, 1, 1000), ("cubic", 1 << 24, 1, 100), ("sphere", 1 << 24, 8, 50), ("sphere", 1 << 26, 8, 50),
          ("rastrigin", 1 << 20, 8, 200), ("sphere", 1 << 20, 2, 500), ("rastrigin", 1 << 20, 32, 300),
          ("cubic", 2048, 1, 100000), ("cubic", 65536, 1, 10000), ("cubic", 32768, 120, 1000), ("cubic", 1024, 1, 1000)]
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["spec", "resident", "wave"]
if len(sys.argv) > 2:  # shape filter: indices into `shapes`
    shapes = [shapes[int(i)] for i in sys.argv[2].split(",")]
for fit, n, d, T in shapes:
    for mode in modes:
        env = dict(os.environ)
        env["CUPSO_SYNC_MODE"] = mode
        for kv in mode.split(":")[1:]:
            k, v = kv.split("=")
            env[k] = v
        env["CUPSO_SYNC_MODE"] = mode.split(":")[0]
        r = subprocess.run([sys.executable, "-c", CODE, fit, str(n), str(d), str(T)], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
        print(f"{fit:9s} n=2^{n.bit_length()-1} d={d} T={T} {mode:22s} {line}", flush=True)
