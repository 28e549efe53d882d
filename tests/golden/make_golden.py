"""Generate tests/golden/reference_runs.json from the UNMODIFIED reference.

Run in the build container (needs /root/reference for oracle/_ref):
    python tests/golden/make_golden.py
Each case records the reference run_serial trace checksum, the per-iteration
gbest particle, the final gbest (fit, particle, pos as hex floats) and the
initial gbest. Cases include the survey's own goldens.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle import Reference, build  # noqa: E402

CASES = [
    # fitness, particles, dims, iters, seed   (first five: SURVEY.md section 8c goldens)
    ("cubic", 1024, 1, 1000, 1),
    ("cubic", 256, 1, 100, 1),
    ("sphere", 1024, 8, 200, 1),
    ("sphere", 1024, 8, 200, 2),
    ("cubic", 128, 120, 50, 1),
    ("rastrigin", 4096, 32, 300, 1),
    ("griewank", 200, 5, 50, 3),
    ("rosenbrock", 300, 4, 60, 4),
    ("rosenbrock", 33, 7, 80, 11),
    ("sphere", 1, 1, 10, 5),
    ("cubic", 33, 120, 100, 22),
    ("sphere", 4097, 3, 120, 9),
] + [("cubic", 1024, 1, 1000, s) for s in range(2, 11)]


def main():
    build(ref=True)
    ref = Reference()
    out = []
    for f, n, d, T, s in CASES:
        r, _ = ref.run("serial", f, n, d, T, s)
        out.append({
            "fitness": f, "particles": n, "dims": d, "iters": T, "seed": s,
            "checksum": ref.checksum(r.trace),
            "trace_particle": [int(x) for x in r.trace_particle],
            "gbest_fit": float(r.gbest_fit).hex(),
            "gbest_particle": int(r.gbest_particle),
            "gbest_pos": [float(x).hex() for x in r.gbest_pos],
            "initial_gbest_fit": float(r.initial_gbest_fit).hex(),
            "trace_last": float(r.trace[-1]).hex(),
        })
        print(f, n, d, T, s, out[-1]["checksum"], r.gbest_particle)
    with open(os.path.join(HERE, "reference_runs.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py (reference run_serial via oracle/_ref)",
                   "cases": out}, fh, indent=1)


if __name__ == "__main__":
    main()
