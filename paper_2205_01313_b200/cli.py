"""pso-bench for the CUDA engines (the reference CLI, tools/pso_bench.cpp:44-156).

    python -m paper_2205_01313_b200.cli --engine cuda-sync --particles 1048576 \
        --dims 1 --iters 1000 --repeat 10 --seed 1 --table
    python -m paper_2205_01313_b200.cli --engine all --sweep 1d --out bench.csv --table
    python -m paper_2205_01313_b200.cli --from-csv bench.csv

Same flags and protocol as the reference (SPEC.md bench-cli): engine
selection ("all" = every CUDA engine), trimmed mean over --repeat runs with
the determinism audit, the frozen CSV schema, the speedup table (baseline
engine --baseline, default cuda-reduction since the reference's "serial" is
the CPU), the paper sweeps (--sweep 1d|120d, --paper-scale), and
--occupancy-out. --device selects the GPU; --devices N shards cuda-sync over N
GPUs of this process (the reference's --devices wish).
"""
from __future__ import annotations

import argparse
import sys

from . import protocol
from .engine import engine_registry, exec_options, find_engine, find_fitness, make_params, rng_key

# bench.hpp:247-265
def sweep_1d(paper_scale: bool):
    iters = 100000 if paper_scale else 1000
    out, n = [], 128
    while n <= 131072:
        out.append((n, iters))
        n *= 2
    return out


def sweep_120d(paper_scale: bool):
    cells = [(128, 5000), (256, 4000), (512, 3000), (1024, 2000), (2048, 2000), (4096, 1500),
             (8192, 1000), (16384, 1000), (32768, 1000), (65536, 1000), (131072, 800)]
    return cells if paper_scale else [(n, min(t, 1000)) for n, t in cells]


def print_record(rec) -> None:
    """pso_bench.cpp:16-22"""
    print(f"{rec.engine:<16s} particles={rec.particles:<7d} dims={rec.dims:<3d} iters={rec.iters:<6d} "
          f"seed={rec.seed:<4d} trimmed_mean={rec.trimmed_mean_seconds():.6f}s "
          f"final_gbest={rec.final_gbest_fit:.17g} checksum={rec.checksum}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pso-bench-cuda",
                                 description="multi-engine particle swarm optimization benchmark (GPU engines)")
    ap.add_argument("--engine", action="append", default=None,
                    help="engine name or 'all' (repeatable); known: all " +
                         " ".join(e.name for e in engine_registry()))
    ap.add_argument("--particles", type=int, default=1024)
    ap.add_argument("--dims", type=int, default=1)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--group-size", type=int, default=128)
    ap.add_argument("--seed", type=int, action="append", default=None)
    ap.add_argument("--repeat", type=int, default=10)
    ap.add_argument("--fitness", default="cubic")
    ap.add_argument("--out", default="bench.csv")
    ap.add_argument("--sweep", choices=["1d", "120d"], default=None)
    ap.add_argument("--paper-scale", action="store_true")
    ap.add_argument("--table", action="store_true", help="print the markdown speedup table")
    ap.add_argument("--csv-table", action="store_true", help="print the table as CSV")
    ap.add_argument("--baseline", default="cuda-reduction", help="engine used as the table's baseline column")
    ap.add_argument("--from-csv", default=None, help="render the table from an existing CSV and exit")
    ap.add_argument("--occupancy-out", default=None, help="write per-iteration queue occupancy (first seed)")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--devices", default=None,
                    help="shard cuda-sync over several GPUs of this process: a count N (GPUs 0..N-1) or a "
                         "comma-separated device list; the trajectory is the single-GPU one")
    a = ap.parse_args(argv)

    if a.from_csv:
        with open(a.from_csv) as fh:
            recs = protocol.read_csv(fh)
        print(protocol.render_table(recs, markdown=not a.csv_table, baseline=a.baseline), end="")
        return 0
    try:
        engines = a.engine or ["cuda-sync"]
        if "all" in engines:
            engines = [e.name for e in engine_registry()]
        for e in engines:
            find_engine(e)  # usage error for unknown names (pso_bench.cpp cli.usage-error)
        find_fitness(a.fitness)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    if a.baseline not in engines:
        engines = [a.baseline] + engines
    devices = None
    if a.devices:
        devices = (tuple(range(int(a.devices))) if "," not in a.devices
                   else tuple(int(x) for x in a.devices.split(",")))
        if len(devices) > 1 and any(e != "cuda-sync" for e in engines if e != a.baseline):
            print("error: --devices shards cuda-sync only", file=sys.stderr)
            return 2
    seeds = a.seed or [1]
    cells = ([(a.particles, a.iters)] if not a.sweep else
             (sweep_1d if a.sweep == "1d" else sweep_120d)(a.paper_scale))
    dims = a.dims if a.sweep != "120d" else 120
    records = []
    for particles, iters in cells:
        for e in engines:
            cfg = protocol.bench_config(engine=e, particles=particles, dims=dims, iters=iters,
                                        group_size=a.group_size, seeds=seeds, repeat=a.repeat,
                                        fitness=a.fitness, out_path=a.out, device=a.device,
                                        devices=devices if e == "cuda-sync" else None)
            for rec in protocol.run_bench(cfg):
                print_record(rec)
                records.append(rec)
    if a.occupancy_out:  # pso_bench.cpp:24-40
        f = find_fitness(a.fitness)
        p = make_params(f, cells[0][0], dims, cells[0][1], a.group_size)
        r = find_engine(engines[-1]).run(p, f, rng_key(seeds[0]), exec_options(device=a.device))
        with open(a.occupancy_out, "w") as fh:
            fh.write("iteration,occupancy\n")
            for t, occ in enumerate(r.queue_occupancy):
                fh.write("%d,%.17g\n" % (t, occ))
    if a.table or a.csv_table:
        print(protocol.render_table(records, markdown=not a.csv_table, baseline=a.baseline), end="")
    return 0


if __name__ == "__main__":
    sys.exit(main())
