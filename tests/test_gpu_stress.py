"""GPU: concurrency stress, the device analogue of the reference's acceptance
criterion 4 (acceptance.cpp:126-200): (a) append uniqueness, (b) lock mutual
exclusion with a counter oracle, (c) queue-lock runs identical across repeats.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_append_uniqueness(cupso):
    """(a) 50 launches x 296 blocks x 200 rounds at random group sizes 2..1024: every
    block-round's claimed slots are exactly 0..n-1 once each, and the grid queue's too."""
    trials, bad = C.c_uint64(), C.c_uint64()
    assert cupso.lib().cupso_selftest_append(0, 50, 4242, C.byref(trials), C.byref(bad)) == 0
    assert trials.value >= 10_000 and bad.value == 0, (trials.value, bad.value)


def test_lock_counter_oracle(cupso):
    """(b) every warp of 4 x SMs blocks increments a plain counter under the spin lock."""
    got, want, lk = C.c_uint64(), C.c_uint64(), C.c_uint32()
    assert cupso.lib().cupso_selftest_lock(0, 50, C.byref(got), C.byref(want), C.byref(lk)) == 0
    assert got.value == want.value and lk.value == 0, (got.value, want.value, lk.value)


def test_queue_lock_repeats_identical_reference_shape(cupso, oracle):
    """(c) the reference's shape (4096 x d=1, 50 iterations, group size 32 -> 128 groups,
    seed 123): 50 repeated queue-lock runs, each bit-identical to run_serial."""
    f = cupso.find_fitness("cubic")
    p = cupso.make_params(f, 4096, 1, 50, 32)
    base = oracle.run_serial("cubic", 4096, 1, 50, 123, want_state=False)
    e = cupso.find_engine("cuda-queue-lock")
    for rep in range(50):
        r = e.run(p, f, cupso.rng_key(123))
        assert np.array_equal(r.trace.view(np.uint64), base.trace.view(np.uint64)), rep
        assert np.array_equal(r.gbest_pos.view(np.uint64), base.gbest_pos.view(np.uint64)), rep


def test_queue_lock_repeats_identical_cfg2(cupso):
    """(c) at BASELINE configs[1] size (2^20 x 1000, group size 32 -> 32768 lock
    contenders per iteration): 50 repeats, each bit-identical to the reference run."""
    path = os.path.join(GOLDEN, "full_cfg2.npz")
    if not os.path.exists(path):
        pytest.skip("full_cfg2.npz missing")
    g = np.load(path)
    f = cupso.find_fitness("cubic")
    p = cupso.make_params(f, 1 << 20, 1, 1000, 32)
    e = cupso.find_engine("cuda-queue-lock")
    for rep in range(50):
        r = e.run(p, f, cupso.rng_key(1))
        assert np.array_equal(r.trace.view(np.uint64), g["trace"].view(np.uint64)), rep
        assert np.array_equal(r.trace_particle, g["trace_particle"]), rep
        assert np.array_equal(r.gbest_pos.view(np.uint64), g["gbest_pos"].view(np.uint64)), rep
