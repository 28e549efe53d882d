"""Run one variant on one shape (for ncu captures): prof_case.py VARIANT FITNESS LOG2N DIMS ITERS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01313_b200 as cp
v, fit, lg, d, T = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
f = cp.find_fitness(fit)
p = cp.make_params(f, 1 << lg, d, T)
with cp.Swarm(p, f, 1) as sw:
    s = sw.step(cp.find_engine(v).variant, T)
    print(f"{v} {fit} 2^{lg} d={d} T={T}: {s*1e6/T:.1f} us/iter")
