"""Generate the full-length BASELINE-shape fixtures tests/golden/full_<case>.npz
from the UNMODIFIED reference (oracle/_ref, the psokit queue-lock engine on all
host threads -- bitwise equal to run_serial, acceptance.cpp:40-76).

Run in the build container (needs /root/reference for oracle/_ref):
    python tests/golden/make_full_golden.py [case ...]

Each fixture holds, for one reference run of the whole T iterations
(engine_serial.hpp:13-44 semantics):
  trace[T], trace_particle[T], occupancy[T]   the per-iteration gbest record
  gbest_fit / gbest_particle / gbest_pos / initial_gbest_fit
  sha256 of every final state array (positions, velocities, fitness, pbest_pos,
  pbest_fit; axis-major soa_index = axis*N + i, swarm.hpp:21-24)
  sample_idx[S] and the final state of those particles (all axes), so a
  tolerance comparison (the cos fitnesses) needs no 100 MB+ fixture.
Consumed by tests/test_gpu_fullsize.py (on the B200; the reference itself does
not travel).
"""
import hashlib
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle import Reference, build  # noqa: E402

# name: (fitness, particles, dims, iters, seed)
CASES = {
    "cfg2": ("cubic", 1 << 20, 1, 1000, 1),        # BASELINE configs[1], full size
    "cfg5proxy": ("sphere", 1 << 24, 8, 50, 1),    # BASELINE configs[4] shape at 2^24 (one shard of 16)
    "cfg5long": ("sphere", 1 << 20, 8, 1000, 3),   # the moving-gbest regime over a long horizon (K ramps to 64)
    "cfg4": ("rastrigin", 1 << 20, 32, 1000, 1),   # BASELINE configs[3], full size
}
ARRAYS = ("positions", "velocities", "fitness", "pbest_pos", "pbest_fit")
SAMPLES = 512


def sample_indices(n: int, gbest_particle: int) -> np.ndarray:
    idx = np.unique(np.concatenate([np.linspace(0, n - 1, SAMPLES).astype(np.int64), [gbest_particle]]))
    return idx.astype(np.int64)


def sampled(arr: np.ndarray, n: int, d: int, idx: np.ndarray) -> np.ndarray:
    """[axis, k] = arr[axis*n + idx[k]] (per-particle arrays: d = 1)."""
    return arr.reshape(d, n)[:, idx].copy()


def make(name: str, ref: Reference) -> None:
    f, n, d, T, seed = CASES[name]
    t0 = time.time()
    r, occ = ref.run("queue-lock", f, n, d, T, seed, threads=0, want_particles=True, want_state=True)
    secs = time.time() - t0
    idx = sample_indices(n, r.gbest_particle)
    out = {
        "fitness": np.array(f), "particles": np.int64(n), "dims": np.int64(d), "iters": np.int64(T),
        "seed": np.uint64(seed),
        "trace": r.trace, "trace_particle": r.trace_particle, "occupancy": occ,
        "gbest_fit": np.float64(r.gbest_fit), "gbest_particle": np.int64(r.gbest_particle),
        "gbest_pos": r.gbest_pos, "initial_gbest_fit": np.float64(r.initial_gbest_fit),
        "checksum": np.array(ref.checksum(r.trace)), "sample_idx": idx,
        "generator": np.array("tests/golden/make_full_golden.py: oracle/_ref queue-lock (unmodified "
                              "reference), all host threads"),
    }
    for k in ARRAYS:
        a = r.state[k]
        out["sha256_" + k] = np.array(hashlib.sha256(a.tobytes()).hexdigest())
        out["sample_" + k] = sampled(a, n, d if k in ("positions", "velocities", "pbest_pos") else 1, idx)
    np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), **out)
    print(f"{name}: {f} n={n} d={d} T={T} seed={seed} gbest={r.gbest_fit!r} @ {r.gbest_particle} "
          f"checksum={out['checksum']} ({secs:.1f} s)", flush=True)


def main():
    build(ref=True)
    ref = Reference()
    for name in (sys.argv[1:] or list(CASES)):
        make(name, ref)


if __name__ == "__main__":
    main()
