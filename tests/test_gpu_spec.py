"""GPU parity of the speculative temporally-blocked cuda-sync mode (k_spec).

A pass runs K iterations per particle in registers against a fixed gbest
snapshot and is re-run exactly when an admission before its last iteration
falsifies that (paper_2205_01313_b200/csrc/cupso_spec.cuh). The bar is the
synchronous one (north star): trace, gbest index trajectory, occupancy and the
full final state bit-identical to run_serial (oracle) / the other synchronous
engines, for every pass length K and however the iterations are chunked.
"""
import os

import numpy as np
import pytest

from test_gpu_parity import BITWISE_FITNESS, assert_bitwise, assert_close, compare_run

pytestmark = pytest.mark.gpu

FITNESS = ["cubic", "sphere", "rosenbrock", "griewank", "rastrigin"]


@pytest.fixture
def spec_env(monkeypatch):
    monkeypatch.setenv("CUPSO_SYNC_MODE", "spec")
    return monkeypatch


def run_sync(cupso, fit, n, d, T, seed, chunks=None):
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, seed) as sw:
        for c in (chunks or [T]):
            sw.step(cupso.SYNC, c)
        mode = sw.sync_mode()
        tr, tp, oc = sw.trace()
        return dict(mode=mode, trace=tr, trace_particle=tp, occupancy=oc, state=sw.state(), gbest=sw.gbest(),
                    stats=sw.spec_stats())


def compare_state(got, orc, fit, what):
    for k in ("positions", "velocities", "pbest_pos", "pbest_fit", "fitness"):
        if fit in BITWISE_FITNESS:
            assert_bitwise(getattr(got, k), orc.state[k], f"{what} {k}")
        else:
            assert_close(getattr(got, k), orc.state[k], f"{what} {k}")


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 8, 12, 16, 32, 64, 120, 256])
@pytest.mark.parametrize("fit", FITNESS)
def test_spec_matches_oracle(cupso, oracle, spec_env, fit, d):
    n, T, seed = (3001, 120, 11) if d <= 120 else (1001, 40, 11)  # odd n: the last unit is part padding
    got = run_sync(cupso, fit, n, d, T, seed)
    assert got["mode"] == "spec"
    orc = oracle.run_serial(fit, n, d, T, seed)

    class R:  # compare_run's shape
        trace, trace_particle = got["trace"], got["trace_particle"]
        gbest_pos, gbest_particle = got["gbest"].pos, got["gbest"].particle
    compare_run(R, orc, fit, f"spec {fit} d={d}")
    compare_state(got["state"], orc, fit, f"spec {fit} d={d}")
    passes, fails, launches = got["stats"]
    assert 0 < passes <= T + fails and launches >= passes


@pytest.mark.parametrize("kmax", ["1", "2", "7", "64"])
def test_spec_pass_length_invariance(cupso, oracle, spec_env, kmax):
    spec_env.setenv("CUPSO_SPEC_K", kmax)
    n, d, T, seed = 5000, 8, 90, 5
    got = run_sync(cupso, "sphere", n, d, T, seed)
    orc = oracle.run_serial("sphere", n, d, T, seed)
    assert_bitwise(got["trace"], orc.trace, f"K={kmax} trace")
    assert np.array_equal(got["trace_particle"], orc.trace_particle)
    compare_state(got["state"], orc, "sphere", f"K={kmax}")
    passes, fails, launches = got["stats"]
    if kmax == "1":
        assert fails == 0 and passes == T  # K = 1 passes are exact by construction
    else:
        assert passes < T + fails


def test_spec_occupancy_matches_queue_engine(cupso, spec_env):
    """queue_occupancy (admitted / N per iteration) equals the classic queue engine's."""
    f = cupso.find_fitness("sphere")
    p = cupso.make_params(f, 4096, 4, 80)
    occ = {}
    for v in (cupso.SYNC, cupso.QUEUE):
        with cupso.Swarm(p, f, 2) as sw:
            sw.step(v, 80)
            tr, tp, oc = sw.trace()
            occ[v] = (tr, tp, oc)
    assert_bitwise(occ[cupso.SYNC][0], occ[cupso.QUEUE][0], "trace")
    assert np.array_equal(occ[cupso.SYNC][1], occ[cupso.QUEUE][1])
    assert_bitwise(occ[cupso.SYNC][2], occ[cupso.QUEUE][2], "occupancy")
    assert occ[cupso.SYNC][2][0] > 0  # iteration 0 admits particles


def test_spec_speculation_is_falsified_and_recovered(cupso, oracle, spec_env):
    """A swarm whose gbest keeps improving: many passes fail and are re-run, result exact."""
    n, d, T, seed = 20000, 2, 200, 3
    got = run_sync(cupso, "rosenbrock", n, d, T, seed)
    passes, fails, launches = got["stats"]
    orc = oracle.run_serial("rosenbrock", n, d, T, seed)
    changes = int(np.count_nonzero(np.diff(orc.trace) != 0))
    assert changes > 3 and fails > 0, (changes, fails)
    assert_bitwise(got["trace"], orc.trace, "trace")
    assert np.array_equal(got["trace_particle"], orc.trace_particle)
    compare_state(got["state"], orc, "rosenbrock", "recovered")


@pytest.mark.parametrize("chunks", [[1] * 12, [5, 7], [3, 1, 8]])
def test_spec_chunked_steps_and_buffer_swap(cupso, oracle, spec_env, chunks):
    """Steps of any length compose; the ping-pong buffer swap is invisible to the caller."""
    n, d, T, seed = 777, 4, 12, 21
    got = run_sync(cupso, "cubic", n, d, T, seed, chunks=chunks)
    orc = oracle.run_serial("cubic", n, d, T, seed)
    assert_bitwise(got["trace"], orc.trace, "trace")
    compare_state(got["state"], orc, "cubic", f"chunks {chunks}")


def test_spec_then_other_variants(cupso, oracle, spec_env):
    """Variants mixed per step after spec passes (graphs re-captured on the swapped buffers)."""
    f = cupso.find_fitness("sphere")
    n, d, T, seed = 1500, 8, 60, 8
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, seed) as sw:
        for v in [cupso.SYNC, cupso.QUEUE_LOCK, cupso.SYNC, cupso.REDUCTION, cupso.SYNC] * 3 + [cupso.SYNC] * 15:
            sw.step(v, 3 if v != cupso.SYNC else 2)
            if sw.iteration >= T:
                break
        if sw.iteration < T:
            sw.step(cupso.SYNC, T - sw.iteration)
        tr, tp, _ = sw.trace()
        st = sw.state()
    orc = oracle.run_serial("sphere", n, d, T, seed)
    assert_bitwise(tr, orc.trace, "trace")
    assert np.array_equal(tp, orc.trace_particle)
    compare_state(st, orc, "sphere", "mixed")


def test_spec_single_particle_and_single_iteration(cupso, oracle, spec_env):
    for n, T in [(1, 40), (2, 1), (3, 17)]:
        got = run_sync(cupso, "sphere", n, 1, T, 9)
        orc = oracle.run_serial("sphere", n, 1, T, 9)
        assert_bitwise(got["trace"], orc.trace, f"n={n} T={T}")
        compare_state(got["state"], orc, "sphere", f"n={n} T={T}")


# The alternative tunings exist only in the exploration build of libcupso.so
# (make -C paper_2205_01313_b200/csrc EXPLORE=1; CUPSO_TEST_EXPLORE=1 runs them).
EXPLORE = os.environ.get("CUPSO_TEST_EXPLORE") == "1"
ALT = pytest.mark.skipif(not EXPLORE, reason="exploration tunings: EXPLORE=1 build only")


@pytest.mark.parametrize("cfg", ["0"] + [pytest.param(c, marks=ALT) for c in "1 2 3 4 5 6 7 8 9 10".split()])
def test_spec_split_tunings_agree(cupso, oracle, monkeypatch, cfg):
    """d = 32 (the cfg4 shape): every lanes-per-particle split of k_spec_split is bit-identical."""
    monkeypatch.setenv("CUPSO_SYNC_MODE", "spec")
    monkeypatch.setenv("CUPSO_SPEC_CFG", cfg)
    n, d, T, seed = 2049, 32, 60, 4
    got = run_sync(cupso, "rastrigin", n, d, T, seed)
    assert got["mode"] == "spec"
    orc = oracle.run_serial("rastrigin", n, d, T, seed)
    assert np.array_equal(got["trace_particle"], orc.trace_particle)
    compare_state(got["state"], orc, "rastrigin", f"cfg {cfg}")
    got_c = run_sync(cupso, "cubic", n, d, T, seed)
    orc_c = oracle.run_serial("cubic", n, d, T, seed)
    assert_bitwise(got_c["trace"], orc_c.trace, "cubic trace")
    compare_state(got_c["state"], orc_c, "cubic", f"cfg {cfg}")


@pytest.mark.parametrize("cfg", ["0"] + [pytest.param(c, marks=ALT) for c in "1 2 3".split()])
@pytest.mark.parametrize("fit", ["rastrigin", "sphere"])
def test_spec_d8_tunings_agree(cupso, oracle, monkeypatch, cfg, fit):
    """d = 8: k_spec at 1-3 blocks/SM and the one-lane split kernel with the
    pbest column in SMEM (the rastrigin default) are bit-identical."""
    monkeypatch.setenv("CUPSO_SYNC_MODE", "spec")
    monkeypatch.setenv("CUPSO_SPEC_CFG", cfg)
    n, d, T, seed = 3001, 8, 80, 6
    got = run_sync(cupso, fit, n, d, T, seed)
    assert got["mode"] == "spec"
    orc = oracle.run_serial(fit, n, d, T, seed)
    assert np.array_equal(got["trace_particle"], orc.trace_particle)
    compare_state(got["state"], orc, fit, f"cfg {cfg}")


def test_spec_cfg5_shape_equals_wave(cupso, monkeypatch):
    """2^22 x d=8 sphere (the cfg5 shape at 1/64 size): spec == wave bitwise, state included."""
    f = cupso.find_fitness("sphere")
    n, d, T = 1 << 22, 8, 24
    p = cupso.make_params(f, n, d, T)
    out = {}
    for mode in ("spec", "wave"):
        monkeypatch.setenv("CUPSO_SYNC_MODE", mode)
        with cupso.Swarm(p, f, 1) as sw:
            sw.step(cupso.SYNC, T)
            assert sw.sync_mode() == mode
            tr, tp, oc = sw.trace()
            st = sw.state()
            out[mode] = (tr, tp, oc, st.positions[::4099].copy(), st.pbest_fit.copy(), sw.spec_stats())
    a, b = out["spec"], out["wave"]
    assert_bitwise(a[0], b[0], "trace")
    assert np.array_equal(a[1], b[1])
    assert_bitwise(a[2], b[2], "occupancy")
    assert_bitwise(a[3], b[3], "positions (strided sample)")
    assert_bitwise(a[4], b[4], "pbest_fit")
    assert a[5][0] < T  # temporally blocked: fewer passes than iterations


@pytest.mark.parametrize("n", [1000, 1 << 16, 1 << 19 + 1])
def test_spec_d1_unit_policy(cupso, oracle, spec_env, n):
    """d = 1: small swarms take one particle per thread, large ones four (float-free
    double2 pairs); every choice stays bit-identical to the oracle."""
    T = 40
    got = run_sync(cupso, "sphere", n, 1, T, 13)
    orc = oracle.run_serial("sphere", n, 1, T, 13, want_state=n < 100000)
    assert_bitwise(got["trace"], orc.trace, f"n={n}")
    assert np.array_equal(got["trace_particle"], orc.trace_particle)
    if n < 100000:
        compare_state(got["state"], orc, "sphere", f"n={n}")


@pytest.mark.parametrize("fit,n,d,T,floor", [("cubic", 1 << 20, 1, 400, 1.0e11), ("sphere", 1 << 22, 8, 24, 1.0e10),
                                             ("cubic", 1 << 16, 1, 2000, 5.0e10)])
def test_spec_throughput_floor(cupso, fit, n, d, T, floor):
    """Regression guard for the kernel choice: the register-resident k_spec runs
    these shapes at 1.6e11 / 1.7e10 / 9.6e10 p-u/s on a B200; a fall-back to a
    slower kernel family (e.g. the ragged split kernel for d = 1) halves that."""
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, 1) as sw:
        best = 1e9
        for _ in range(2):
            sw.init()
            best = min(best, sw.step(cupso.SYNC, T))
        assert sw.sync_mode() == "spec"
    assert n * T / best > floor, f"{n * T / best:.3e} p-u/s"


def test_spec_needs_exact_draw_scaling(cupso):
    """A cognitive / social factor whose 2^-53 scaling would underflow (|c| < 2^-969)
    keeps cuda-sync off the register kernels (vel_step53 would not be exact);
    the other modes still match the reduction engine bit for bit."""
    f = cupso.find_fitness("sphere")
    base = cupso.make_params(f, 2000, 4, 30)
    p = cupso.pso_params(**{**base.__dict__, "cognitive": 1e-300}) if hasattr(base, "__dict__") else None
    if p is None:
        pytest.skip("pso_params is not a plain record")
    out = {}
    for v in (cupso.SYNC, cupso.REDUCTION):
        with cupso.Swarm(p, f, 4) as sw:
            sw.step(v, 30)
            out[v] = sw.trace()[0]
            if v == cupso.SYNC:
                assert sw.sync_mode() != "spec"
    assert_bitwise(out[cupso.SYNC], out[cupso.REDUCTION], "trace")


@pytest.mark.parametrize("seed", [0, 2**32, 2**64 - 1])
def test_spec_extreme_seeds(cupso, oracle, spec_env, seed):
    """Philox key = the 64-bit seed split in halves (rng.hpp:22-30): the edges of the key space."""
    got = run_sync(cupso, "sphere", 1537, 8, 50, seed)
    orc = oracle.run_serial("sphere", 1537, 8, 50, seed)
    assert_bitwise(got["trace"], orc.trace, f"seed {seed}")
    compare_state(got["state"], orc, "sphere", f"seed {seed}")


def test_async_throughput_floor(cupso):
    """Regression guard for cuda-async's register kernel (1.9e11 p-u/s at 2^24 x d=1 on a B200)."""
    f = cupso.find_fitness("cubic")
    p = cupso.make_params(f, 1 << 24, 1, 60)
    with cupso.Swarm(p, f, 1) as sw:
        s = sw.step(cupso.ASYNC, 60)
        assert sw.async_mode() == "reg"
    assert (1 << 24) * 60 / s > 1.2e11, f"{(1 << 24) * 60 / s:.3e} p-u/s"


@pytest.mark.parametrize("n,d,want", [(32768, 120, "spec"), (65536, 120, "wave"), (70000, 100, "wave"),
                                      (1 << 20, 64, "spec"), (1 << 17, 256, "wave")])
def test_wide_swarm_mode_choice(cupso, n, d, want):
    """Above 64 dims the pass kernel runs only for swarms below 65536 particles:
    larger ones are faster as one k_wave launch per iteration."""
    f = cupso.find_fitness("sphere")
    p = cupso.make_params(f, n, d, 2)
    with cupso.Swarm(p, f, 3) as sw:
        sw.step(cupso.SYNC, 2)
        assert sw.sync_mode() == want


@pytest.mark.parametrize("fit,d", [("rastrigin", 32), ("sphere", 12), ("griewank", 100), ("rosenbrock", 64),
                                   ("cubic", 256), ("sphere", 3)])
def test_async_split_kernel_invariants(cupso, oracle, fit, d):
    """cuda-async above 8 dims (and at 3/5/6/7) runs k_async_split (registers, G lanes per
    particle): monotone trace, a self-consistent gbest record equal to the best pbest."""
    f = cupso.find_fitness(fit)
    n, T = 3001, 70
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, 5) as sw:
        sw.step(cupso.ASYNC, 30)
        sw.step(cupso.ASYNC, T - 30)
        assert sw.async_mode() == "reg"
        tr, _, _ = sw.trace()
        gb = sw.gbest()
        st = sw.state()
    assert (np.diff(tr) >= 0).all() and tr[-1] == gb.fit
    assert st.pbest_fit.max() == gb.fit and st.pbest_fit[gb.particle] == gb.fit
    pos = st.pbest_pos.reshape(d, n)[:, gb.particle]
    assert np.array_equal(pos.view(np.uint64), np.asarray(gb.pos).view(np.uint64))
    want = oracle.fitness(fit, gb.pos)
    assert abs(want - gb.fit) <= 1e-12 * max(1.0, abs(want))
    assert (st.positions >= p.min_pos).all() and (st.positions <= p.max_pos).all()


@pytest.mark.parametrize("fit,n,d", [("cubic", 934003, 1), ("sphere", 1048576, 1), ("rosenbrock", 308105, 2),
                                     ("sphere", 606209, 1)])
def test_spec_tail_round_matches_oracle(cupso, oracle, spec_env, fit, n, d):
    """k_spec's last grid round in half-size units (3 rounds of 4 particles + 1
    of 2 at 2^20 d = 1 on 148 SMs): the tail units, their ragged end and the
    main/tail boundary stay bit-identical to run_serial."""
    T, seed = 40, 23
    got = run_sync(cupso, fit, n, d, T, seed)
    assert got["mode"] == "spec"
    orc = oracle.run_serial(fit, n, d, T, seed)

    class R:
        trace, trace_particle = got["trace"], got["trace_particle"]
        gbest_pos, gbest_particle = got["gbest"].pos, got["gbest"].particle
    compare_run(R, orc, fit, f"tail {fit} n={n} d={d}")
    compare_state(got["state"], orc, fit, f"tail {fit} n={n}")
