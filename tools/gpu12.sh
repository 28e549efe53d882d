timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches and sync or golden or final_state or acceptance_cross" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "cfg2 or ragged or modes" 2>&1 | tail -2
python - <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2205_01313_b200 as cp
f = cp.find_fitness("cubic"); p = cp.make_params(f, 1 << 20, 1, 1000)
with cp.Swarm(p, f, 1) as sw:
    best = 1e9
    for _ in range(5):
        sw.init(); best = min(best, sw.step(cp.SYNC, 1000))
    print("cfg2 mode", sw.sync_mode(), "grid", sw.sync_grid_blocks(), f"{best*1e3:.3f} ms/1000 it -> {2**20*1000/best:.3e} p-u/s")
PY
