"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Bar (north star): synchronous variants bit-match the reference gbest
trajectory -- trace, per-iteration gbest index, final gbest position, and the
full final swarm state -- for cubic / sphere / rosenbrock. For the cos-based
fitness functions (griewank, harness rastrigin) CUDA's cos may differ from
glibc's by an ulp, so there the gbest index trajectory must match exactly and
fitness / positions agree within REL_TOL = 1e-5 relative (north star).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # north-star tolerance for cos-based fitness (fitness and positions)
BITWISE_FITNESS = {"cubic", "sphere", "rosenbrock"}
DET_ENGINES = ["cuda-reduction", "cuda-unrolled", "cuda-queue", "cuda-queue-lock", "cuda-sync"]
HERE = os.path.dirname(os.path.abspath(__file__))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, what
    bad = np.nonzero(bits(a) != bits(b))[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: {a[bad[:3]]} vs {b[bad[:3]]}"


def assert_close(a, b, what, rel=REL_TOL):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    np.testing.assert_allclose(a, b, rtol=rel, atol=rel * 1e-3, err_msg=what)


def compare_run(res, orc, fitness, what, state=None):
    if fitness in BITWISE_FITNESS:
        assert_bitwise(res.trace, orc.trace, what + " trace")
        assert_bitwise(res.gbest_pos, orc.gbest_pos, what + " gbest_pos")
    else:
        assert_close(res.trace, orc.trace, what + " trace")
        assert_close(res.gbest_pos, orc.gbest_pos, what + " gbest_pos")
    assert np.array_equal(res.trace_particle, orc.trace_particle), what + " gbest index trajectory"
    assert res.gbest_particle == orc.gbest_particle, what + " gbest_particle"


# ---------------------------------------------------------------- primitives
def test_philox_kats_on_device(cupso):
    import ctypes as C
    L = cupso.lib()
    ctr = np.array([[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344]],
                   dtype=np.uint32)
    key = np.array([[0, 0], [0xFFFFFFFF, 0xFFFFFFFF], [0xa4093822, 0x299f31d0]], dtype=np.uint32)
    out = np.zeros((3, 4), dtype=np.uint32)
    P = C.POINTER(C.c_uint32)
    assert L.cupso_philox_batch(0, ctr.ctypes.data_as(P), key.ctypes.data_as(P), out.ctypes.data_as(P), 3) == 0
    # test_rng.cpp:18-23
    assert [hex(x) for x in out[0]] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(x) for x in out[1]] == ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(x) for x in out[2]] == ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


def test_uniform01_matches_oracle(cupso, oracle):
    import ctypes as C
    rng = np.random.default_rng(7)
    n = 4096
    draws = rng.integers(0, 2**32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    draws[:, 3] %= 4
    seed = 0x9E3779B97F4A7C15
    out = np.zeros(n)
    assert cupso.lib().cupso_uniform01_batch(0, seed, draws.ctypes.data_as(C.POINTER(C.c_uint32)),
                                             out.ctypes.data_as(C.POINTER(C.c_double)), n) == 0
    want = np.array([oracle.uniform01(seed, *map(int, d)) for d in draws])
    assert_bitwise(out, want, "uniform01")
    assert (out >= 0).all() and (out < 1).all()


@pytest.mark.parametrize("name", ["cubic", "sphere", "rosenbrock", "griewank", "rastrigin"])
def test_fitness_on_device(cupso, oracle, name):
    f = cupso.find_fitness(name)
    rng = np.random.default_rng(3)
    for d in (1, 2, 7, 32):
        x = rng.uniform(f.lo, f.hi, size=(d, 257))
        got = f.eval_batch(x)
        want = np.array([oracle.fitness(name, x[:, i]) for i in range(x.shape[1])])
        if name in BITWISE_FITNESS:
            assert_bitwise(got, want, f"{name} d={d}")
        else:
            np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-12)


def test_fitness_pins_on_device(cupso):
    # test_fitness.cpp:15-23, 44-58
    cubic = cupso.find_fitness("cubic")
    for d in (1, 7):
        assert cubic(np.zeros(d)) == 8000.0 * d
    assert cubic([100.0]) == 900000.0
    assert cubic([-100.0]) == -900000.0
    assert cupso.find_fitness("sphere")(np.zeros(6)) == 0.0
    assert cupso.find_fitness("griewank")(np.zeros(6)) == 0.0
    assert cupso.find_fitness("rosenbrock")(np.ones(6)) == 0.0
    for n in ("sphere", "griewank", "rosenbrock"):
        assert cupso.find_fitness(n)(np.full(6, 0.25)) < 0.0
    with pytest.raises(cupso.DomainError):
        cubic([101.0])
    with pytest.raises(cupso.DomainError):
        cubic([float("nan")])


def test_kinematics_pins_on_device(cupso, oracle):
    # test_swarm.cpp:102-141
    import ctypes as C
    L = cupso.lib()

    def kin(p, v, x, pb, g, r1, r2):
        arr = [np.array([a], np.float64) for a in (v, x, pb, g, r1, r2)]
        vo, xo = np.zeros(1), np.zeros(1)
        dp = C.POINTER(C.c_double)
        cp = p.to_c()
        assert L.cupso_eval_kinematics(0, C.byref(cp), *[a.ctypes.data_as(dp) for a in arr],
                                       vo.ctypes.data_as(dp), xo.ctypes.data_as(dp), 1) == 0
        return vo[0], xo[0]

    p = cupso.pso_params(particle_cnt=1, dims=1, max_iter=1)
    assert kin(p, 7.0, 5.0, 5.0, 5.0, 0.3, 0.9)[0] == 7.0
    p2 = cupso.pso_params(particle_cnt=1, dims=1, max_iter=1, inertia=0.5)
    assert kin(p2, 10.0, 0.0, 3.0, 4.0, 0.0, 0.0)[0] == 5.0
    assert kin(p, 0.0, 0.0, 1.0, 2.0, 0.5, 0.5)[0] == 3.0
    p3 = cupso.pso_params(particle_cnt=1, dims=1, max_iter=1, max_v=2.5)
    assert kin(p3, 0.0, 0.0, 1.0, 2.0, 0.5, 0.5)[0] == 2.5
    # position_step pins: v' = 0 -> x; 99 + 5 -> 100; -100 - 1 -> -100
    assert kin(cupso.pso_params(min_v=0.0, max_v=0.0), 0.0, 42.0, 42.0, 42.0, 0.0, 0.0)[1] == 42.0
    assert kin(cupso.pso_params(min_v=5.0, max_v=5.0), 5.0, 99.0, 99.0, 99.0, 0.0, 0.0)[1] == 100.0
    assert kin(cupso.pso_params(min_v=-1.0, max_v=-1.0), -1.0, -100.0, -100.0, -100.0, 0.0, 0.0)[1] == -100.0
    # random cases vs the oracle, incl. saturation both ways
    rng = np.random.default_rng(11)
    op = oracle.make_params("cubic", 4, 1, 1)
    pp = cupso.pso_params(min_pos=op.min_pos, max_pos=op.max_pos, min_v=op.min_v, max_v=op.max_v)
    for _ in range(200):
        v, x, pb, g = rng.uniform(-150, 150, 4)
        r1, r2 = rng.uniform(0, 1, 2)
        vo, xo = kin(pp, v, x, pb, g, r1, r2)
        wv = oracle.velocity_step(v, x, pb, g, op, r1, r2)
        assert bits(vo) == bits(wv)
        assert bits(xo) == bits(oracle.position_step(x, wv, op))


# ----------------------------------------------------------------------- init
@pytest.mark.parametrize("fitness,n,d,seed", [("cubic", 33, 1, 1), ("cubic", 128, 120, 0xfeed),
                                              ("sphere", 1000, 8, 3), ("rastrigin", 257, 32, 4),
                                              ("rosenbrock", 1, 5, 9)])
def test_init_matches_oracle(cupso, oracle, fitness, n, d, seed):
    f = cupso.find_fitness(fitness)
    p = cupso.make_params(f, n, d, 1)
    with cupso.Swarm(p, f, seed) as sw:
        s = sw.state()
        gf, gi = sw.initial_gbest()
        gb = sw.gbest()
    st, of, oi, op = oracle.init(fitness, n, d, seed)
    assert_bitwise(s.positions, st["positions"], "init positions")
    assert_bitwise(s.velocities, st["velocities"], "init velocities")
    assert_bitwise(s.pbest_pos, st["positions"], "init pbest_pos")
    if fitness in BITWISE_FITNESS:
        assert_bitwise(s.pbest_fit, st["pbest_fit"], "init pbest_fit")
        assert_bitwise(s.fitness, st["fitness"], "init fitness")
        assert gf == of
    else:
        assert_close(s.pbest_fit, st["pbest_fit"], "init pbest_fit", rel=1e-12)
    assert gi == oi and gb.particle == oi
    assert_bitwise(gb.pos, op, "init gbest pos")


# ------------------------------------------------------------- engine parity
CASES = [
    ("cubic", 1024, 1, 200, 1, 128),
    ("cubic", 33, 120, 60, 22, 32),
    ("sphere", 1024, 8, 200, 1, 128),
    ("sphere", 4097, 3, 120, 9, 64),
    ("rosenbrock", 300, 4, 60, 4, 128),
    ("rosenbrock", 33, 7, 80, 11, 32),
    ("griewank", 200, 5, 50, 3, 128),
    ("rastrigin", 2048, 32, 100, 1, 128),
    ("sphere", 1, 1, 10, 5, 128),
    ("cubic", 300, 2, 30, 9, 48),     # non-power-of-two group (looped-tree fallback)
]


@pytest.mark.parametrize("engine", DET_ENGINES)
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_engine_matches_serial(cupso, oracle, engine, case):
    fitness, n, d, T, seed, gs = case
    f = cupso.find_fitness(fitness)
    p = cupso.make_params(f, n, d, T, gs)
    res = cupso.find_engine(engine).run(p, f, cupso.rng_key(seed))
    orc = oracle.run_serial(fitness, n, d, T, seed, params=oracle.make_params(fitness, n, d, T, gs))
    compare_run(res, orc, fitness, f"{engine} {case}")
    assert len(res.trace) == T
    assert res.initial_gbest_fit == orc.initial_gbest_fit or fitness not in BITWISE_FITNESS
    if engine in ("cuda-reduction", "cuda-unrolled"):
        assert res.queue_occupancy.size == 0  # reference reduction logs no occupancy
    else:
        assert res.queue_occupancy.size == T
        assert ((res.queue_occupancy >= 0) & (res.queue_occupancy <= 1)).all()


@pytest.mark.parametrize("engine", DET_ENGINES)
def test_final_state_bitwise(cupso, oracle, engine):
    fitness, n, d, T, seed = "sphere", 777, 6, 90, 13
    f = cupso.find_fitness(fitness)
    p = cupso.make_params(f, n, d, T, 64)
    variant = cupso.find_engine(engine).variant
    with cupso.Swarm(p, f, seed) as sw:
        sw.step(variant, T)
        s = sw.state()
    orc = oracle.run_serial(fitness, n, d, T, seed, params=oracle.make_params(fitness, n, d, T, 64))
    for k in ("positions", "velocities", "fitness", "pbest_pos", "pbest_fit"):
        assert_bitwise(getattr(s, k), orc.state[k], f"{engine} final {k}")


def test_golden_reference_runs(cupso):
    """Goldens generated from the unmodified reference (tests/golden/make_golden.py)."""
    with open(os.path.join(HERE, "golden", "reference_runs.json")) as fh:
        cases = json.load(fh)["cases"]
    for c in cases:
        f = cupso.find_fitness(c["fitness"])
        p = cupso.make_params(f, c["particles"], c["dims"], c["iters"])
        res = cupso.find_engine("cuda-sync").run(p, f, cupso.rng_key(c["seed"]))
        what = f"golden {c['fitness']} {c['particles']}x{c['dims']}x{c['iters']} seed {c['seed']}"
        assert list(map(int, res.trace_particle)) == c["trace_particle"], what
        assert res.gbest_particle == c["gbest_particle"], what
        if c["fitness"] in BITWISE_FITNESS:
            assert cupso.trace_checksum(res.trace) == c["checksum"], what
            assert [float(x).hex() for x in res.gbest_pos] == c["gbest_pos"], what
            assert float(res.gbest_fit).hex() == c["gbest_fit"], what
        else:
            assert abs(res.gbest_fit - float.fromhex(c["gbest_fit"])) <= REL_TOL * abs(float.fromhex(c["gbest_fit"]))


# ---------------------------------------------------- acceptance criteria
def test_acceptance_cross_engine_equivalence(cupso, oracle):
    """acceptance.cpp:40-76 for the CUDA engines, the reference's 5 seeds (acceptance.cpp:47)."""
    f = cupso.find_fitness("cubic")
    runs = 0
    for n in (33, 128, 256, 1024):
        for d in (1, 120):
            for seed in (11, 22, 33, 44, 55):
                base = oracle.run_serial("cubic", n, d, 100, seed, want_state=False)
                for gs in (32, 128):
                    p = cupso.make_params(f, n, d, 100, gs)
                    for e in DET_ENGINES:
                        r = cupso.find_engine(e).run(p, f, cupso.rng_key(seed))
                        assert_bitwise(r.trace, base.trace, f"{e} n={n} d={d} gs={gs} seed={seed}")
                        assert_bitwise(r.gbest_pos, base.gbest_pos, f"{e} gbest_pos")
                        runs += 1
    assert runs == 4 * 2 * 5 * 2 * len(DET_ENGINES)


@pytest.mark.parametrize("engine", DET_ENGINES + ["cuda-async"])
def test_acceptance_per_iteration_oracle(cupso, oracle, engine):
    """acceptance.cpp:79-105: gbest(t) = max(gbest(t-1), max_i recomputed fit_i(t))."""
    f = cupso.find_fitness("cubic")
    for d in (1, 3):
        p = cupso.make_params(f, 256, d, 50, 64)
        _, init_fit, _, _ = oracle.init("cubic", 256, d, 101 + d)
        prev = [init_fit]
        violations = []

        def obs(t, s, gb):
            best = max(oracle.fitness("cubic", s.positions[i::s.particle_cnt]) for i in range(s.particle_cnt))
            if gb.fit != max(prev[0], best):
                violations.append(t)
            prev[0] = gb.fit

        cupso.find_engine(engine).run(p, f, cupso.rng_key(101 + d), None, obs)
        assert not violations, f"{engine} d={d}: {violations[:5]}"


@pytest.mark.parametrize("engine", DET_ENGINES + ["cuda-async"])
def test_acceptance_convergence_1d_cubic(cupso, engine):
    """acceptance.cpp:108-124: >= 9/10 seeds reach 899999."""
    f = cupso.find_fitness("cubic")
    p = cupso.make_params(f, 1024, 1, 1000, 128)
    hits = sum(cupso.find_engine(engine).run(p, f, cupso.rng_key(s)).gbest_fit >= 899999.0
               for s in range(1, 11))
    assert hits >= 9
