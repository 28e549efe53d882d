"""GPU: randomised parity soak of the synchronous engines against the oracle.

Each trial draws a fitness with an exact (cos-free) fitness, a particle count,
a dimension (1..256, so every kernel family is hit: k_spec, the split kernels
ragged or not, the wave / persistent fallbacks past 256 are covered
elsewhere), a 64-bit seed, a pass-length cap (CUPSO_SPEC_K) and a random
chunking of the iterations with a random deterministic engine per chunk
(cuda-sync, reduction, unrolled, queue, queue-lock). The trace, the gbest index
trajectory and the final state must equal run_serial bit for bit
(engine_serial.hpp:13-44). FUZZ_TRIALS (default 12), FUZZ_SEED and FUZZ_CELLS size a run.
"""
import os

import numpy as np
import pytest

from test_gpu_parity import assert_bitwise

pytestmark = pytest.mark.gpu

TRIALS = int(os.environ.get("FUZZ_TRIALS", "12"))
BASE = int(os.environ.get("FUZZ_SEED", "20261017"))
CELLS = int(os.environ.get("FUZZ_CELLS", "200000"))  # bounds n * d * 40 of the exact-fitness trials


def draw_case(rng):
    fit = rng.choice(["cubic", "sphere", "rosenbrock"])
    d = int(rng.choice([1, 1, 2, 3, 4, 5, 7, 8, 8, 9, 12, 16, 17, 31, 32, 33, 64, 100, 129, 256]))
    n = int(rng.integers(1, max(2, CELLS // (d * 40))))
    T = int(rng.integers(1, 90))
    seed = int(rng.integers(0, 2**64 - 1, dtype=np.uint64))
    kmax = str(rng.choice([1, 2, 3, 5, 16, 64]))
    cuts = sorted(set(int(x) for x in rng.integers(1, T, size=int(rng.integers(0, 4))))) if T > 1 else []
    bounds = [0] + cuts + [T]
    chunks = [b - a for a, b in zip(bounds, bounds[1:]) if b > a]
    engines = [str(rng.choice(["cuda-sync", "cuda-sync", "cuda-reduction", "cuda-unrolled", "cuda-queue",
                               "cuda-queue-lock"])) for _ in chunks]
    return fit, n, d, T, seed, kmax, chunks, engines


@pytest.mark.parametrize("trial", range(TRIALS))
def test_fuzz_sync_engines_match_serial(cupso, oracle, monkeypatch, trial):
    rng = np.random.default_rng(BASE + trial)
    fit, n, d, T, seed, kmax, chunks, engines = draw_case(rng)
    what = f"{fit} n={n} d={d} T={T} seed={seed} K<={kmax} chunks={chunks} engines={engines}"
    monkeypatch.setenv("CUPSO_SPEC_K", kmax)
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, seed) as sw:
        for c, e in zip(chunks, engines):
            sw.step(cupso.find_engine(e).variant, c)
        tr, tp, _ = sw.trace()
        st = sw.state()
    orc = oracle.run_serial(fit, n, d, T, seed)
    assert_bitwise(tr, orc.trace, f"{what}: trace")
    assert np.array_equal(tp, orc.trace_particle), f"{what}: gbest index trajectory"
    for k in ("positions", "velocities", "pbest_pos", "pbest_fit", "fitness"):
        assert_bitwise(getattr(st, k), orc.state[k], f"{what}: {k}")


SHARD_TRIALS = int(os.environ.get("FUZZ_SHARD_TRIALS", "4"))


@pytest.mark.parametrize("trial", range(SHARD_TRIALS))
def test_fuzz_shards_match_single_swarm(cupso, monkeypatch, trial):
    """Random shard counts (2-4) of random swarms, host-thread all-gather or the
    in-kernel peer-memory exchange, random chunking: every shard's trace and
    gbest index trajectory equal the single swarm's, and the concatenated shard
    positions equal its state, bit for bit."""
    import threading

    from test_gpu_scale import _ThreadAllGather, same
    rng = np.random.default_rng(BASE + 10_000 + trial)
    fit = str(rng.choice(["cubic", "sphere", "rosenbrock"]))
    d = int(rng.choice([1, 2, 4, 5, 8, 12, 32, 64]))
    shards = int(rng.integers(2, 5))
    n = int(rng.integers(shards, max(shards + 1, 120_000 // (d * 20))))
    T = int(rng.integers(2, 70))
    seed = int(rng.integers(0, 2**63))
    p2p = bool(rng.integers(0, 2))
    monkeypatch.setenv("CUPSO_SPEC_K", str(rng.choice([2, 8, 64])))
    cut = int(rng.integers(1, T))
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, seed) as whole:
        whole.step(cupso.SYNC, T)
        wtr, wtp, _ = whole.trace()
        wst = whole.state()
    parts = [cupso.Swarm(p, f, seed, first=a, count=c, init=False)
             for a, c in (cupso.shard_range(n, shards, r) for r in range(shards))]
    what = f"{fit} n={n} d={d} T={T} shards={shards} p2p={p2p} cut={cut}"
    try:
        cupso.init_shards(parts)
        if p2p:
            cupso.p2p_shards(parts)
        ag = _ThreadAllGather(shards)
        errs = []

        def run(r):
            try:
                for c in (cut, T - cut):
                    if p2p:
                        parts[r].step(cupso.SYNC, c)
                    else:
                        parts[r].step_exchange(c, shards, lambda loc: ag(r, loc))
            except Exception as e:  # pragma: no cover - reported below
                errs.append(e)

        th = [threading.Thread(target=run, args=(r,)) for r in range(shards)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        assert not errs, (what, errs)
        for sh in parts:
            tr, tp, _ = sh.trace()
            assert same(tr, wtr) and np.array_equal(tp, wtp), what
        pos = np.concatenate([sh.state().positions.reshape(d, -1) for sh in parts], axis=1)
        assert same(pos.reshape(-1), wst.positions), what
    finally:
        for sh in parts:
            sh.close()


STAT_TRIALS = int(os.environ.get("FUZZ_STAT_TRIALS", "6"))


@pytest.mark.parametrize("trial", range(STAT_TRIALS))
def test_fuzz_statistical_engines_invariants(cupso, oracle, monkeypatch, trial):
    """cuda-async (every schedule) and cuda-sync-f32 on random shapes, any
    fitness: a monotone trace ending at the gbest; the gbest record is a
    consistent (fitness, position) pair that equals the best pbest (at FP32 for
    the FP32 engine); the state stays in the box."""
    rng = np.random.default_rng(BASE + 20_000 + trial)
    fit = str(rng.choice(["cubic", "sphere", "rosenbrock", "griewank", "rastrigin"]))
    d = int(rng.choice([1, 2, 3, 4, 8, 9, 16, 32, 33, 100, 256]))
    n = int(rng.integers(1, max(2, 150_000 // (d * 20))))
    T = int(rng.integers(2, 60))
    seed = int(rng.integers(0, 2**63))
    engine = str(rng.choice(["cuda-async", "cuda-sync-f32"]))
    if engine == "cuda-async":
        monkeypatch.setenv("CUPSO_ASYNC_MODE", str(rng.choice(["reg", "tiled", "plain"])))
        monkeypatch.setenv("CUPSO_ASYNC_K", str(rng.choice([1, 5, 32])))
    what = f"{engine} {fit} n={n} d={d} T={T} seed={seed}"
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, n, d, T)
    cut = int(rng.integers(1, T))
    with cupso.Swarm(p, f, seed) as sw:
        init_fit = sw.initial_gbest()[0]
        for c in (cut, T - cut):
            sw.step(cupso.find_engine(engine).variant, c)
        tr, tp, occ = sw.trace()
        gb = sw.gbest()
        st = sw.state()
    assert (np.diff(tr) >= 0).all() and tr[0] >= init_fit, what
    assert tr[-1] == gb.fit and 0 <= gb.particle < n, what
    assert ((occ >= 0) & (occ <= 1)).all(), what
    rel = 1e-4 if engine == "cuda-sync-f32" else 1e-9
    assert abs(oracle.fitness(fit, gb.pos) - gb.fit) <= rel * max(1.0, abs(gb.fit)), what
    if engine == "cuda-sync-f32":
        assert np.float32(gb.fit) == np.float32(st.pbest_fit.max()), what
        assert (np.abs(st.positions) <= np.float32(f.hi)).all(), what
    else:
        assert gb.fit == st.pbest_fit.max(), what
        assert (np.abs(st.positions) <= f.hi).all(), what


COS_TRIALS = int(os.environ.get("FUZZ_COS_TRIALS", "3"))


@pytest.mark.parametrize("trial", range(COS_TRIALS))
def test_fuzz_cos_fitness_sync_close_to_serial(cupso, oracle, monkeypatch, trial):
    """griewank / rastrigin through cuda-sync: the device cos is within 2 ulp of
    glibc's, not bitwise (section 2), so the trace and the state are compared at
    the cos tolerance -- a gbest race decided by that last ulp would show up here."""
    from test_gpu_parity import assert_close
    rng = np.random.default_rng(BASE + 30_000 + trial)
    fit = str(rng.choice(["griewank", "rastrigin"]))
    d = int(rng.choice([1, 2, 3, 4, 8, 12, 16, 32, 64]))
    n = int(rng.integers(1, max(2, 60_000 // (d * 20))))
    T = int(rng.integers(1, 60))
    seed = int(rng.integers(0, 2**63))
    what = f"{fit} n={n} d={d} T={T} seed={seed}"
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, seed) as sw:
        sw.step(cupso.SYNC, T)
        tr, tp, _ = sw.trace()
        st = sw.state()
    orc = oracle.run_serial(fit, n, d, T, seed)
    assert np.array_equal(tp, orc.trace_particle), f"{what}: gbest index trajectory"
    assert_close(tr, orc.trace, f"{what}: trace")
    assert_close(st.positions, orc.state["positions"], f"{what}: positions")
