"""GPU: the statistical engines against run_serial's distribution (north_star:
"The asynchronous variant is checked statistically, comparing final fitness
across 32 seeds").

cuda-async (free-running blocks, lock-free CAS-published gbest) and
cuda-sync-f32 (FP32 state, its own RNG stream) are not bitwise reproductions
of run_serial, so their final-fitness distributions over 32 seeds are compared
with run_serial's on non-degenerate fitnesses (sphere d=8, Rastrigin d=32; the
1-D cubic hits 900000 at iteration 0 for every seed and cannot discriminate).
run_serial's distribution is produced by cuda-sync, which is bitwise
run_serial (tests/test_gpu_parity.py, tests/test_gpu_fullsize.py) -- checked
again here on the oracle for two seeds. Bar: a two-sided Mann-Whitney U test
does not reject equality at ALPHA, and the median costs are within RATIO.

cuda-async is nondeterministic (free-running blocks), so its p-value changes
from run to run; on Rastrigin d=32 it also converges slightly differently by
design (a particle may move against a gbest found by a block that is further
ahead): five B200 runs gave p = 0.05-0.19 with median cost ratios 1.03-1.05.
Its gate is therefore ALPHA_ASYNC = 0.001 (a false failure at round end would
otherwise be a few-percent event) together with the same RATIO bound; the
deterministic cuda-sync-f32 keeps ALPHA = 0.01.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEEDS = range(1, 33)
ALPHA = 0.01
ALPHA_ASYNC = 0.001
RATIO = 1.5
N, T = 4096, 300


def final_costs(cupso, engine, fitness, d):
    f = cupso.find_fitness(fitness)
    p = cupso.make_params(f, N, d, T)
    e = cupso.find_engine(engine)
    return np.array([-e.run(p, f, cupso.rng_key(s)).gbest_fit for s in SEEDS])


@pytest.fixture(scope="module")
def serial_costs(cupso, oracle):
    out = {}
    for fitness, d in (("sphere", 8), ("rastrigin", 32)):
        c = final_costs(cupso, "cuda-sync", fitness, d)
        for s in (1, 2):  # cuda-sync is run_serial, bit for bit (cos fitness: within 1e-5)
            o = oracle.run_serial(fitness, N, d, T, s, want_state=False)
            assert abs(-o.gbest_fit - c[s - 1]) <= 1e-5 * abs(o.gbest_fit)
        out[fitness] = c
    return out


@pytest.mark.parametrize("engine", ["cuda-async", "cuda-sync-f32"])
@pytest.mark.parametrize("fitness,d", [("sphere", 8), ("rastrigin", 32)])
def test_final_fitness_distribution_matches_run_serial(cupso, serial_costs, engine, fitness, d):
    from scipy.stats import mannwhitneyu
    base = serial_costs[fitness]
    got = final_costs(cupso, engine, fitness, d)
    assert np.isfinite(got).all() and (got >= 0).all()
    p = mannwhitneyu(got, base, alternative="two-sided").pvalue
    ratio = np.median(got) / np.median(base)
    print(f"{engine} {fitness} d={d}: median {np.median(got):.5g} vs run_serial {np.median(base):.5g} "
          f"(ratio {ratio:.3f}), Mann-Whitney p={p:.3f}")
    assert p > (ALPHA_ASYNC if engine == "cuda-async" else ALPHA), (p, ratio)
    assert 1 / RATIO <= ratio <= RATIO, (p, ratio)
