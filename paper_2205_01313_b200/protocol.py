"""The reference's bench protocol (psokit bench.hpp) for the CUDA engines.

Same trimmed mean, FNV-1a trace checksum, determinism audit, frozen CSV
schema and speedup table, so CPU-reference rows and CUDA rows share one table
(SURVEY.md section 8(f) "next" item 1).
"""
from __future__ import annotations

import io
import os
import struct
from dataclasses import dataclass, field
from typing import Iterable, Optional

from .engine import exec_options, find_engine, find_fitness, make_params, rng_key


def trimmed_mean(xs) -> float:
    """bench.hpp:20-28: mean after dropping exactly one min and one max."""
    xs = list(xs)
    if len(xs) < 3:
        raise ValueError("trimmed_mean: need at least 3 samples to drop min and max")
    s = sorted(xs)
    total = 0.0
    for v in s[1:-1]:
        total += v
    return total / (len(s) - 2)


def trace_checksum(trace) -> str:
    """bench.hpp:31-44: FNV-1a over the exact bit patterns; 16 hex digits."""
    h = 1469598103934665603
    for v in trace:
        bits = struct.unpack("<Q", struct.pack("<d", float(v)))[0]
        for _ in range(8):
            h ^= bits & 0xFF
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
            bits >>= 8
    return f"{h:016x}"


@dataclass
class bench_config:
    """bench.hpp:46-66 defaults."""
    engine: str = "cuda-sync"
    particles: int = 1024
    dims: int = 1
    iters: int = 1000
    group_size: int = 128
    seeds: list = field(default_factory=lambda: [1])
    repeat: int = 10
    fitness: str = "cubic"
    out_path: str = ""
    device: int = 0
    devices: Optional[tuple] = None  # cuda-sync sharded over these GPUs (exec_options.devices)

    def validate(self) -> None:
        if self.repeat < 3:
            raise ValueError("bench_config: repeat must be >= 3 (the trimmed mean drops one min and one max)")
        if not self.seeds:
            raise ValueError("bench_config: need at least one seed")
        find_engine(self.engine)
        find_fitness(self.fitness)


@dataclass
class bench_record:
    """bench.hpp:70-81."""
    engine: str
    particles: int = 0
    dims: int = 1
    iters: int = 1
    seed: int = 1
    seconds: list = field(default_factory=list)
    final_gbest_fit: float = 0.0
    checksum: str = ""

    def trimmed_mean_seconds(self) -> float:
        return trimmed_mean(self.seconds)


csv_header = "engine,particles,dims,iters,seed,run_idx,seconds,final_gbest_fit,trace_checksum"


def _g17(v: float) -> str:
    return "%.17g" % v


def write_csv_row(out, rec: bench_record, run_idx: int) -> None:
    """bench.hpp:86-94."""
    out.write(f"{rec.engine},{rec.particles},{rec.dims},{rec.iters},{rec.seed},{run_idx},"
              f"{_g17(rec.seconds[run_idx])},{_g17(rec.final_gbest_fit)},{rec.checksum}\n")


def run_bench(cfg: bench_config) -> list[bench_record]:
    """bench.hpp:99-141: repeat runs per seed, checksum audit, CSV rows.
    Times are device seconds of the iteration loop (CUDA events)."""
    cfg.validate()
    engine = find_engine(cfg.engine)
    f = find_fitness(cfg.fitness)
    p = make_params(f, cfg.particles, cfg.dims, cfg.iters, cfg.group_size)
    opts = exec_options(device=cfg.device, devices=cfg.devices)
    csv = None
    if cfg.out_path:
        fresh = not os.path.exists(cfg.out_path)
        csv = open(cfg.out_path, "a")
        if fresh:
            csv.write(csv_header + "\n")
    records = []
    try:
        for seed in cfg.seeds:
            rec = bench_record(cfg.engine, cfg.particles, cfg.dims, cfg.iters, seed)
            for run in range(cfg.repeat):
                res = engine.run(p, f, rng_key(seed), opts, None)
                rec.seconds.append(res.compute_seconds)
                s = trace_checksum(res.trace)
                if run == 0:
                    rec.final_gbest_fit = res.gbest_fit
                    rec.checksum = s
                elif s != rec.checksum and engine.deterministic:
                    raise RuntimeError(f"determinism violation: engine {cfg.engine} seed {seed} "
                                       "produced differing traces")
                if csv:
                    write_csv_row(csv, rec, run)
            records.append(rec)
    finally:
        if csv:
            csv.close()
    return records


def read_csv(stream: io.TextIOBase) -> list[bench_record]:
    """bench.hpp:145-185 (inverse of write_csv_row)."""
    lines = stream.read().splitlines()
    if not lines or lines[0] != csv_header:
        raise RuntimeError("bad CSV: missing or unexpected header")
    cells: dict = {}
    order = []
    for line in lines[1:]:
        if not line:
            continue
        cols = line.split(",")
        if len(cols) != 9:
            raise RuntimeError("bad CSV row: " + line)
        key = (cols[0], int(cols[1]), int(cols[2]), int(cols[3]), int(cols[4]))
        if key not in cells:
            cells[key] = bench_record(cols[0], key[1], key[2], key[3], key[4], [],
                                      float(cols[7]), cols[8])
            order.append(key)
        cell = cells[key]
        if len(cell.seconds) != int(cols[5]):
            raise RuntimeError("bad CSV: run_idx out of order in " + line)
        cell.seconds.append(float(cols[6]))
    return [cells[k] for k in order]


def render_table(records: Iterable[bench_record], markdown: bool = True,
                 baseline: str = "serial") -> str:
    """bench.hpp:191-238: one row per (cell, engine), speedup = baseline / engine."""
    base_sum: dict = {}
    base_cnt: dict = {}
    engines: dict = {}
    for rec in records:
        key = (rec.particles, rec.dims, rec.iters)
        if rec.engine == baseline:
            base_sum[key] = base_sum.get(key, 0.0) + rec.trimmed_mean_seconds()
            base_cnt[key] = base_cnt.get(key, 0) + 1
        else:
            slot = engines.setdefault(key, {}).setdefault(rec.engine, [0.0, 0])
            slot[0] += rec.trimmed_mean_seconds()
            slot[1] += 1
    out = ("| engine | particles | dims | iters | serial (s) | engine (s) | speedup |\n"
           "|---|---:|---:|---:|---:|---:|---:|\n") if markdown else \
        "engine,particles,dims,iters,serial_seconds,engine_seconds,speedup\n"
    for key in sorted(engines):
        particles, dims, iters = key
        if key not in base_cnt:
            raise ValueError(f"render_table: no serial baseline for particles={particles} "
                             f"dims={dims} iters={iters}")
        serial_s = base_sum[key] / base_cnt[key]
        rows = sorted(((n, s[0] / s[1]) for n, s in engines[key].items()), key=lambda r: r[1])
        for name, es in rows:
            if markdown:
                out += (f"| {name} | {particles} | {dims} | {iters} | {serial_s:.3f} | {es:.3f} | "
                        f"{serial_s / es:.2f} |\n")
            else:
                out += f"{name},{particles},{dims},{iters},{serial_s:.3f},{es:.3f},{serial_s / es:.2f}\n"
    return out
