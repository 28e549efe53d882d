"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01313_b200 as cp

CASES = [  # (fitness, n, d, T, variant, env)
    ("sphere", 3001, 1, 40, cp.SYNC, {"CUPSO_SYNC_MODE": "spec"}),
    ("rosenbrock", 2001, 8, 30, cp.SYNC, {"CUPSO_SYNC_MODE": "spec"}),
    ("rastrigin", 1001, 32, 20, cp.SYNC, {"CUPSO_SYNC_MODE": "spec"}),
    ("griewank", 777, 12, 20, cp.SYNC, {"CUPSO_SYNC_MODE": "spec"}),
    ("cubic", 4097, 4, 40, cp.ASYNC, {"CUPSO_ASYNC_MODE": "reg"}),
    ("sphere", 3001, 8, 30, cp.SYNC_F32, {}),
    ("sphere", 3001, 3, 10, cp.SYNC_F32, {}),
    ("sphere", 3001, 6, 10, cp.SYNC, {"CUPSO_SYNC_MODE": "wave"}),
    ("cubic", 5000, 1, 20, cp.SYNC, {"CUPSO_SYNC_MODE": "resident"}),
    ("cubic", 5000, 2, 10, cp.QUEUE_LOCK, {}),
    ("cubic", 5000, 2, 10, cp.REDUCTION, {}),
    ("rosenbrock", 2001, 17, 20, cp.SYNC_F32, {}),   # k_spec32_split, ragged
    ("rastrigin", 1001, 32, 20, cp.SYNC_F32, {}),    # k_spec32_split 8 x 4
    ("griewank", 999, 300, 5, cp.SYNC_F32, {}),      # k_wave32 (d > 256)
    ("cubic", 700001, 1, 5, cp.SYNC, {"CUPSO_SYNC_MODE": "spec"}),   # k_spec NP=4 + the NP=2 tail round
    ("sphere", 300001, 2, 5, cp.SYNC, {"CUPSO_SYNC_MODE": "spec"}),  # k_spec NP=2 + the NP=1 tail round
    ("griewank", 777, 12, 20, cp.ASYNC, {"CUPSO_ASYNC_MODE": "reg"}),  # k_async_split, ragged
]
which = sys.argv[1:] and [int(x) for x in sys.argv[1].split(",")] or range(len(CASES))
for k in which:
    fit, n, d, T, v, env = CASES[k]
    os.environ.update(env)
    f = cp.find_fitness(fit)
    p = cp.make_params(f, n, d, T)
    with cp.Swarm(p, f, 3) as sw:
        sw.step(v, T)
        print(k, fit, n, d, T, cp.lib().cupso_variant_name(v).decode(), env, "gbest", sw.gbest().fit, flush=True)
    for key in env:
        del os.environ[key]
