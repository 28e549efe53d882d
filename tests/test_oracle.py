"""CPU: pin the oracle (the checker) before trusting it.

1. The reference's own known-answer vectors (test_rng.cpp:18-23,
   test_fitness.cpp:15-58, test_swarm.cpp:102-141).
2. Bitwise agreement with the UNMODIFIED reference compiled from
   /root/reference (oracle/_ref, built by oracle/Makefile) where available.
3. The committed golden fixtures generated from that reference
   (tests/golden/make_golden.py) -- these need no /root/reference.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
KATS = [  # test_rng.cpp:18-23
    ((0, 0, 0, 0), 0, 0, (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xFFFFFFFF,) * 4, 0xFFFFFFFF, 0xFFFFFFFF, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), 0xa4093822, 0x299f31d0,
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("ctr,k0,k1,want", KATS)
def test_philox_kats(oracle, ctr, k0, k1, want):
    assert oracle.philox(ctr, k0, k1) == want


def test_uniform01_properties(oracle):
    key = 0x9E3779B97F4A7C15
    vals = np.array([oracle.uniform01(key, 0, i, 0, 0) for i in range(20000)])
    assert (vals >= 0).all() and (vals < 1).all()
    assert abs(vals.mean() - 0.5) < 0.01
    bins = np.histogram(vals, bins=16, range=(0, 1))[0]
    exp = len(vals) / 16
    assert ((bins - exp) ** 2 / exp).sum() < 37.697  # test_rng.cpp:54-71
    # slot separation (test_rng.cpp:44-52)
    r2 = np.array([oracle.uniform01(key, 0, i, 0, 1) for i in range(20000)])
    assert not np.any(vals == r2)


def test_fitness_pins(oracle):
    for d in (1, 7):
        assert oracle.fitness("cubic", np.zeros(d)) == 8000.0 * d
    assert oracle.fitness("cubic", [100.0]) == 900000.0
    assert oracle.fitness("cubic", [-100.0]) == -900000.0
    assert oracle.fitness("sphere", np.zeros(6)) == 0.0
    assert oracle.fitness("griewank", np.zeros(6)) == 0.0
    assert oracle.fitness("rosenbrock", np.ones(6)) == 0.0
    assert oracle.fitness("rastrigin", np.zeros(6)) == 0.0
    for n in ("sphere", "griewank", "rosenbrock", "rastrigin"):
        assert oracle.fitness(n, np.full(6, 0.25)) < 0.0


def test_kinematics_pins(oracle):
    p = oracle.make_params("cubic", 1, 1, 1)
    p.min_v, p.max_v = -100.0, 100.0
    assert oracle.velocity_step(7.0, 5.0, 5.0, 5.0, p, 0.3, 0.9) == 7.0
    p.inertia = 0.5
    assert oracle.velocity_step(10.0, 0.0, 3.0, 4.0, p, 0.0, 0.0) == 5.0
    p.inertia = 1.0
    assert oracle.velocity_step(0.0, 0.0, 1.0, 2.0, p, 0.5, 0.5) == 3.0
    p.max_v = 2.5
    assert oracle.velocity_step(0.0, 0.0, 1.0, 2.0, p, 0.5, 0.5) == 2.5
    assert oracle.position_step(42.0, 0.0, p) == 42.0
    assert oracle.position_step(99.0, 5.0, p) == 100.0
    assert oracle.position_step(-100.0, -1.0, p) == -100.0


def test_params_validation_messages(oracle):
    with pytest.raises(ValueError, match="particle_cnt"):
        oracle.make_params("cubic", 0, 1, 1)
    with pytest.raises(ValueError, match="dims"):
        oracle.make_params("cubic", 1, 0, 1)
    with pytest.raises(ValueError, match="max_iter"):
        oracle.make_params("cubic", 1, 1, 0)
    with pytest.raises(ValueError, match="group_size"):
        oracle.make_params("cubic", 1, 1, 1, 0)


def test_trimmed_mean_and_checksum(oracle):
    assert oracle.trimmed_mean([1.0, 2.0, 3.0]) == 2.0
    assert np.isnan(oracle.trimmed_mean([1.0, 2.0]))
    assert oracle.checksum(np.array([900000.0] * 1000)) == "585d124f8e33b353"


def test_golden_fixtures_reproduced_by_oracle(oracle):
    with open(os.path.join(HERE, "golden", "reference_runs.json")) as fh:
        cases = json.load(fh)["cases"]
    assert len(cases) >= 12
    for c in cases:
        if c["particles"] * c["dims"] * c["iters"] > 3_000_000:
            continue  # keep the CPU suite fast; the big ones are covered on the GPU
        r = oracle.run_serial(c["fitness"], c["particles"], c["dims"], c["iters"], c["seed"], want_state=False)
        what = f"{c['fitness']} {c['particles']}x{c['dims']}x{c['iters']} seed {c['seed']}"
        assert oracle.checksum(r.trace) == c["checksum"], what
        assert list(map(int, r.trace_particle)) == c["trace_particle"], what
        assert float(r.gbest_fit).hex() == c["gbest_fit"], what
        assert [float(x).hex() for x in r.gbest_pos] == c["gbest_pos"], what
        assert float(r.initial_gbest_fit).hex() == c["initial_gbest_fit"], what


# ----------------------------------------------------- against the reference
def test_reference_kats(reference):
    for ctr, k0, k1, want in KATS:
        assert reference.philox(ctr, k0, k1) == want


def test_oracle_matches_reference_primitives(oracle, reference):
    rng = np.random.default_rng(5)
    for name in ("cubic", "sphere", "rosenbrock", "griewank", "rastrigin"):
        lo, hi = {"rosenbrock": (-2.048, 2.048), "griewank": (-600, 600),
                  "rastrigin": (-5.12, 5.12)}.get(name, (-100, 100))
        for d in (1, 3, 32):
            for _ in range(20):
                x = rng.uniform(lo, hi, d)
                assert bits(oracle.fitness(name, x)) == bits(reference.fitness(name, x)), name


@pytest.mark.parametrize("case", [("cubic", 256, 1, 100, 1), ("sphere", 500, 8, 60, 2),
                                  ("rosenbrock", 33, 7, 80, 11), ("griewank", 200, 5, 50, 3),
                                  ("rastrigin", 300, 16, 40, 4), ("cubic", 130, 120, 20, 12)])
def test_oracle_matches_reference_runs(oracle, reference, case):
    f, n, d, T, s = case
    a = oracle.run_serial(f, n, d, T, s)
    b, _ = reference.run("serial", f, n, d, T, s, want_state=True)
    assert np.array_equal(bits(a.trace), bits(b.trace))
    assert np.array_equal(a.trace_particle, b.trace_particle)
    assert np.array_equal(bits(a.gbest_pos), bits(b.gbest_pos))
    for k in a.state:
        assert np.array_equal(bits(a.state[k]), bits(b.state[k])), k


def test_reference_parallel_engines_equal_serial(reference):
    """The reference's own cross-engine claim holds in this build (acceptance.cpp:40-76)."""
    base, _ = reference.run("serial", "cubic", 300, 2, 30, 9, group_size=32)
    for e in ("reduction", "unrolled", "queue", "queue-lock"):
        r, occ = reference.run(e, "cubic", 300, 2, 30, 9, group_size=32, threads=4)
        assert np.array_equal(bits(r.trace), bits(base.trace)), e
        assert np.array_equal(bits(r.gbest_pos), bits(base.gbest_pos)), e


def test_reference_rejects_bad_params(reference):
    with pytest.raises(ValueError, match="particle_cnt"):
        reference.run("serial", "cubic", 0, 1, 1, 1)
    with pytest.raises(ValueError, match="unknown engine"):
        reference.run("warpspeed", "cubic", 8, 1, 1, 1)


def test_oracle_shard_step_replays_serial(oracle):
    """Two shards advanced with the snapshot + candidate exchange reproduce
    run_serial -- the protocol the multi-GPU path uses."""
    f, n, d, T, seed = "sphere", 301, 4, 40, 17
    p = oracle.make_params(f, n, d, T)
    st, gfit, gidx, gpos = oracle.init(f, n, d, seed)
    trace = []
    for t in range(T):
        snap_pos, snap_fit = gpos.copy(), gfit
        recs = [oracle.shard_step(f, p, seed, t, st, a, b - a, snap_pos, snap_fit)
                for a, b in ((0, 150), (150, n))]
        best = None
        for bf, bi, bp, _ in recs:
            if bi == 0xFFFFFFFF:
                continue
            if best is None or bf > best[0] or (bf == best[0] and bi < best[1]):
                best = (bf, bi, bp)
        if best is not None and best[0] > snap_fit:
            gfit, gidx, gpos = best
        trace.append(gfit)
    ref = oracle.run_serial(f, n, d, T, seed)
    assert np.array_equal(bits(trace), bits(ref.trace))
    assert np.array_equal(bits(gpos), bits(ref.gbest_pos))


@pytest.mark.parametrize("case", ["cfg2", "cfg5proxy", "cfg5long", "cfg4"])
def test_full_size_fixtures_consistent(oracle, case):
    """The full-length reference fixtures (tests/golden/make_full_golden.py) are
    self-consistent, and the cfg2 one carries the survey's own checksum."""
    path = os.path.join(HERE, "golden", f"full_{case}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = np.load(path)
    n, d, T = int(g["particles"]), int(g["dims"]), int(g["iters"])
    tr = g["trace"]
    assert tr.shape == (T,) and g["trace_particle"].shape == (T,)
    assert (np.diff(tr) >= 0).all() and tr[-1] == g["gbest_fit"]
    assert g["trace_particle"][-1] == g["gbest_particle"]
    assert oracle.checksum(tr) == str(g["checksum"])
    # the gbest particle is in the sample: its pbest is the gbest record
    k = int(np.nonzero(g["sample_idx"] == g["gbest_particle"])[0][0])
    assert g["sample_pbest_fit"][0, k] == g["gbest_fit"]
    assert bits(g["sample_pbest_pos"][:, k]).tolist() == bits(g["gbest_pos"]).tolist()
    # sampled particles' stored fitness is the oracle's fitness of their position
    fit = str(g["fitness"])
    for j in range(0, len(g["sample_idx"]), 97):
        got = oracle.fitness(fit, g["sample_positions"][:, j])
        want = g["sample_fitness"][0, j]
        assert got == want if fit != "rastrigin" else abs(got - want) <= 1e-12 * max(1.0, abs(want))
    if case == "cfg2":
        assert str(g["checksum"]) == "585d124f8e33b353"  # SURVEY.md 8c, seed 1 at N=1024 and N=2^20 alike
        assert n == 1 << 20 and d == 1 and T == 1000
