"""B200-native cuPSO (arXiv 2205.01313): the per-iteration PSO step on sm_100a.

The package mirrors the reference psokit solver API (pso_params, make_params,
find_fitness, engine_registry, find_engine, run_result, ...) on top of
libcupso.so, whose C-ABI is declared in include/cupso.h. Importing the package
does not require a GPU; running an engine does (no CPU fallback).
"""
from ._lib import (ASYNC, QUEUE, QUEUE_LOCK, REDUCTION, SYNC, SYNC_F32, UNROLLED, CupsoError, DomainError,
                   LogicError, lib)
from .engine import (FIT_SENTINEL, NO_PARTICLE, device_count, engine_entry, engine_registry,
                     exec_options, find_engine, find_fitness, fitness_fn, fitness_registry,
                     global_best, make_params, pso_params, rng_key, run_cuda, run_result,
                     swarm_state)
from .protocol import (bench_config, bench_record, csv_header, read_csv, render_table, run_bench,
                       trace_checksum, trimmed_mean, write_csv_row)
from .swarm import (Swarm, decode_record, encode_record, init_shards, link_shards, nccl_unique_id, p2p_shards, select_winner,
                    shard_range, step_shards)

__all__ = [n for n in dir() if not n.startswith("_")]
