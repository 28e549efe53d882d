"""GPU: the FP32 engine cuda-sync-f32.

FP32 state with float4 rows, one Philox call per particle-axis, FMA
kinematics, and the paper's packed 64-bit (fitness, index) atomicMax
aggregation. Not bitwise against the FP64 reference: checked statistically
(final fitness over 32 seeds against run_serial, tests/test_gpu_stats.py) and
by invariants.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fit,d", [("cubic", 1), ("sphere", 8), ("rastrigin", 2), ("rosenbrock", 4),
                                   ("griewank", 3), ("sphere", 5), ("rastrigin", 32), ("rosenbrock", 17),
                                   ("griewank", 100), ("cubic", 256), ("sphere", 300)])
def test_f32_invariants(cupso, oracle, fit, d):
    """Monotone trace; the record is a consistent (fit, pos) pair of an FP32
    particle; gbest = max pbest; state in the box. d = 3 / 5 / 17 / 32 / 100 /
    256 run k_spec32_split (ragged but for 32), d = 300 k_wave32."""
    f = cupso.find_fitness(fit)
    n, T = 5001, 90
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, 7) as sw:
        sw.step(cupso.SYNC_F32, 40)
        sw.step(cupso.SYNC_F32, T - 40)
        tr, tp, occ = sw.trace()
        gb = sw.gbest()
        st = sw.state()
        init_fit = sw.initial_gbest()[0]
    assert (np.diff(tr) >= 0).all() and tr[0] >= init_fit
    assert tr[-1] == gb.fit and tp[-1] == gb.particle
    assert gb.fit == st.pbest_fit.max()
    holder = gb.particle
    pb = st.pbest_pos.reshape(d, n)[:, holder]
    assert np.array_equal(pb.astype(np.float32).astype(np.float64), pb)  # an FP32 state
    assert np.array_equal(pb, gb.pos)
    assert abs(oracle.fitness(fit, gb.pos) - gb.fit) <= 1e-4 * max(1.0, abs(gb.fit))
    assert (np.abs(st.positions) <= np.float32(f.hi)).all()  # the FP32 box (bounds rounded to FP32)
    assert ((occ >= 0) & (occ <= 1)).all()


def test_f32_cfg2_shape_converges(cupso):
    f = cupso.find_fitness("cubic")
    p = cupso.make_params(f, 1 << 20, 1, 200)
    r = cupso.find_engine("cuda-sync-f32").run(p, f, cupso.rng_key(1))
    assert r.gbest_fit == 900000.0 and len(r.trace) == 200


def test_f32_then_fp64_engines(cupso):
    """Switching engines converts the state (FP32 -> FP64) transparently."""
    f = cupso.find_fitness("sphere")
    p = cupso.make_params(f, 3000, 8, 60)
    with cupso.Swarm(p, f, 3) as sw:
        sw.step(cupso.SYNC_F32, 20)
        sw.step(cupso.SYNC, 20)
        sw.step(cupso.SYNC_F32, 10)
        sw.step(cupso.QUEUE_LOCK, 10)
        tr, _, _ = sw.trace()
        st = sw.state()
        gb = sw.gbest()
    assert (np.diff(tr) >= 0).all() and gb.fit == st.pbest_fit.max()


@pytest.mark.parametrize("fit,d", [("rastrigin", 32), ("rosenbrock", 17)])
def test_f32_wide_statistics(cupso, fit, d):
    """The split FP32 kernel (lanes' partial fitnesses combined by a butterfly)
    optimises like the FP64 engine: median final fitness over 12 seeds."""
    f = cupso.find_fitness(fit)
    p = cupso.make_params(f, 8192, d, 200)
    sync = np.array([cupso.find_engine("cuda-sync").run(p, f, cupso.rng_key(s)).gbest_fit for s in range(1, 13)])
    f32 = np.array([cupso.find_engine("cuda-sync-f32").run(p, f, cupso.rng_key(s)).gbest_fit for s in range(1, 13)])
    med_s, med_f = np.median(-sync), np.median(-f32)
    assert med_f < 1.5 * med_s, (med_f, med_s)


def test_f32_wide_uses_pass_kernel(cupso):
    """d = 32 runs register-resident passes (a handful of launches for 256
    iterations), not one k_wave32 launch per iteration."""
    f = cupso.find_fitness("rastrigin")
    p = cupso.make_params(f, 1 << 16, 32, 256)
    with cupso.Swarm(p, f, 1) as sw:
        sw.step(cupso.SYNC_F32, 256)
        passes, fails, launches = sw.spec_stats()
    assert 0 < launches < 128, (passes, fails, launches)


@pytest.mark.parametrize("n,d", [(1, 9), (7, 31), (33, 64), (130, 129)])
def test_f32_split_ragged_edges(cupso, n, d):
    """Tiny / ragged swarms on the split kernel: partial lane groups at the
    swarm's end and partially filled axis slots keep the engine's invariants."""
    f = cupso.find_fitness("sphere")
    T = 30
    p = cupso.make_params(f, n, d, T)
    with cupso.Swarm(p, f, 11) as sw:
        sw.step(cupso.SYNC_F32, T)
        tr, tp, _ = sw.trace()
        gb = sw.gbest()
        st = sw.state()
    assert (np.diff(tr) >= 0).all() and tr[-1] == gb.fit and 0 <= gb.particle < n
    # a swarm this small may see no admission in T iterations: the gbest record
    # is then still the FP64 one from init_swarm, and the FP32 state holds its
    # FP32 rounding -- so compare at FP32
    f32 = np.float32
    assert f32(gb.fit) == f32(st.pbest_fit.max())
    assert np.array_equal(st.pbest_pos.reshape(d, n)[:, gb.particle].astype(f32), gb.pos.astype(f32))
    assert abs(-float(np.sum(gb.pos.astype(np.float64) ** 2)) - gb.fit) <= 1e-4 * max(1.0, abs(gb.fit))
    assert (np.abs(st.positions) <= np.float32(f.hi)).all()
