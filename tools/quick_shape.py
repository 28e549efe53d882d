"""Device time of cuda-sync on one shape (exploration): quick_shape.py FITNESS N D T -> p-u/s."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01313_b200 as cp
fit, n, d, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
f = cp.find_fitness(fit)
p = cp.make_params(f, n, d, T)
with cp.Swarm(p, f, 1) as sw:
    best = 1e9
    for rep in range(3):
        sw.init()
        best = min(best, sw.step(cp.SYNC, T))
    print(json.dumps(dict(fit=fit, n=n, d=d, T=T, pus=n * T / best, mode=sw.sync_mode(), gbest=sw.gbest().fit)))
