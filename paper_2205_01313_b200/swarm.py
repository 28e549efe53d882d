"""Device-resident swarm handle (per-iteration drop-in, checkpoint/resume, shards).

Wraps the cupso_swarm handle API of include/cupso.h. One handle = one swarm
(or one shard of a multi-GPU swarm) in HBM plus its stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib
from .engine import (NO_PARTICLE, fitness_fn, global_best, pso_params, rng_key, swarm_state,
                     _dp, _up)


class Swarm:
    """A swarm (or shard [first, first+count)) resident on one GPU."""

    def __init__(self, p: pso_params, f: fitness_fn, key: rng_key | int, device: int = 0,
                 first: int = 0, count: Optional[int] = None, init: bool = True):
        p.validate()
        self.params = p
        self.fitness = f
        self.seed = key.seed if isinstance(key, rng_key) else int(key)
        self.device = device
        self.first = first
        self.count = p.particle_cnt - first if count is None else count
        self._cp = p.to_c()
        h = C.c_void_p()
        check(lib().cupso_create_shard(C.byref(self._cp), f.id, self.seed & (2**64 - 1), device,
                                       first, self.count, C.byref(h)))
        self._h = h
        if init:
            self.init()

    # -- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().cupso_destroy(self._h)
            self._h = None

    def __del__(self):  # best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- stepping --------------------------------------------------------------
    def init(self) -> None:
        check(lib().cupso_init(self._h))

    def step(self, variant: int, iters: int = 1) -> float:
        """Advance `iters` iterations; returns their device seconds (CUDA events)."""
        s = C.c_double()
        check(lib().cupso_step(self._h, variant, iters, C.byref(s)))
        return s.value

    @property
    def iteration(self) -> int:
        return lib().cupso_iteration(self._h)

    def synchronize(self) -> None:
        check(lib().cupso_synchronize(self._h))

    # -- results -----------------------------------------------------------------
    def gbest(self) -> global_best:
        f = C.c_double()
        i = C.c_uint32()
        pos = np.zeros(self.params.dims)
        check(lib().cupso_get_gbest(self._h, C.byref(f), C.byref(i), _dp(pos)))
        return global_best(f.value, pos, i.value)

    def initial_gbest(self) -> tuple[float, int]:
        f = C.c_double()
        i = C.c_uint32()
        check(lib().cupso_get_initial_gbest(self._h, C.byref(f), C.byref(i)))
        return f.value, i.value

    def trace(self, first: int = 0, count: Optional[int] = None):
        count = self.iteration - first if count is None else count
        tr = np.zeros(count)
        tp = np.zeros(count, dtype=np.uint32)
        oc = np.zeros(count)
        check(lib().cupso_get_trace(self._h, first, count, _dp(tr), _up(tp), _dp(oc)))
        return tr, tp, oc

    def state(self) -> swarm_state:
        n, d = self.count, self.params.dims
        a = {k: np.zeros(n * d) for k in ("positions", "velocities", "pbest_pos")}
        a.update({k: np.zeros(n) for k in ("fitness", "pbest_fit")})
        check(lib().cupso_download_state(self._h, _dp(a["positions"]), _dp(a["velocities"]),
                                         _dp(a["fitness"]), _dp(a["pbest_pos"]),
                                         _dp(a["pbest_fit"])))
        return swarm_state(n, d, a["positions"], a["velocities"], a["fitness"], a["pbest_pos"],
                           a["pbest_fit"])

    def load_state(self, iteration: int, s: swarm_state, gb: global_best) -> None:
        """Checkpoint resume: the counter-based RNG makes (state, t, seed) sufficient."""
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in
                (s.positions, s.velocities, s.pbest_pos, s.pbest_fit, gb.pos)]
        check(lib().cupso_upload_state(self._h, iteration, _dp(arrs[0]), _dp(arrs[1]),
                                       _dp(arrs[2]), _dp(arrs[3]), gb.fit,
                                       gb.particle & 0xFFFFFFFF, _dp(arrs[4])))

    def device_bytes(self) -> int:
        return lib().cupso_device_bytes(self._h)

    def sync_grid_blocks(self) -> int:
        return lib().cupso_sync_grid_blocks(self._h)

    SYNC_MODES = {0: "undecided", 1: "persistent", 2: "wave", 3: "resident", 4: "nccl-sharded", 5: "spec", 6: "nccl-sharded-spec"}

    def sync_mode(self) -> str:
        return self.SYNC_MODES[lib().cupso_sync_mode(self._h)]

    def spec_stats(self) -> tuple[int, int, int]:
        """(passes, falsified passes, launches) of the speculative cuda-sync mode on this handle."""
        a, b, c = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        check(lib().cupso_spec_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    ASYNC_MODES = {0: "undecided", 1: "plain", 2: "tiled", 3: "reg"}

    def async_mode(self) -> str:
        return self.ASYNC_MODES[lib().cupso_async_mode(self._h)]

    def stream(self) -> int:
        return lib().cupso_stream(self._h) or 0

    # -- shard exchange (multi-GPU) ------------------------------------------------
    @property
    def record_bytes(self) -> int:
        return lib().cupso_record_bytes(self.params.dims)

    def snapshot_record(self) -> bytes:
        buf = C.create_string_buffer(self.record_bytes)
        check(lib().cupso_shard_snapshot(self._h, buf))
        return buf.raw

    def adopt(self, records: list[bytes] | bytes) -> None:
        blob = records if isinstance(records, (bytes, bytearray)) else b"".join(records)
        buf = C.create_string_buffer(bytes(blob), len(blob))
        check(lib().cupso_shard_adopt(self._h, buf, len(blob) // self.record_bytes))

    def propose(self) -> bytes:
        buf = C.create_string_buffer(self.record_bytes)
        check(lib().cupso_shard_propose(self._h, buf))
        return buf.raw

    def commit(self, records: list[bytes] | bytes) -> None:
        blob = records if isinstance(records, (bytes, bytearray)) else b"".join(records)
        n = len(blob) // self.record_bytes
        buf = C.create_string_buffer(bytes(blob), len(blob))
        check(lib().cupso_shard_commit(self._h, buf, n))

    def step_exchange(self, iters: int, nranks: int, allgather) -> float:
        """cuda-sync steps of a host-exchanged shard: allgather(local: bytes) -> list of
        nranks records (bytes, rank order). Called once per speculative pass (or per
        iteration where no speculative kernel exists); every shard must step alike."""
        err = []

        def cb(local, allp, nbytes, _user):
            try:
                recs = allgather(C.string_at(local, nbytes))
                blob = b"".join(recs)
                assert len(blob) == nbytes * nranks
                C.memmove(allp, blob, len(blob))
                return 0
            except Exception as e:  # surfaced after the call returns
                err.append(e)
                return 1

        fn = _lib.EXCHANGE_FN(cb)
        s = C.c_double()
        st = lib().cupso_step_exchange(self._h, iters, nranks, fn, None, C.byref(s))
        if err:
            raise err[0]
        check(st)
        return s.value

    IPC_RECORD = 192  # bytes per rank of cupso_ipc_handles

    def ipc_handles(self, nranks: int, p2p: bool) -> bytes:
        """This shard's CUDA IPC exports for shards in other processes (cupso_ipc_handles)."""
        buf = C.create_string_buffer(self.IPC_RECORD)
        check(lib().cupso_ipc_handles(self._h, nranks, int(p2p), buf))
        return buf.raw

    def ipc_link(self, all_handles: list[bytes], rank: int, p2p: bool) -> None:
        """Open the other ranks' exports (rank order): early-stop hints, and with p2p the
        pass-record exchange fused into the pass kernel (then step with plain step())."""
        blob = b"".join(all_handles)
        check(lib().cupso_ipc_link(self._h, blob, len(all_handles), rank, int(p2p)))

    def nccl_init(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().cupso_nccl_init(self._h, buf, nranks, rank))


def link_shards(shards: list["Swarm"]) -> None:
    """Shards of one swarm in this process: a falsified speculative pass on one
    stops the others early (cupso_shard_link; results never depend on it)."""
    arr = (C.c_void_p * len(shards))(*[sh._h for sh in shards])
    check(lib().cupso_shard_link(arr, len(shards)))


def p2p_shards(shards: list["Swarm"]) -> None:
    """Shards of one swarm in this process exchange their pass records inside the
    pass kernel over peer memory (cupso_shard_p2p). Step each from its own thread."""
    arr = (C.c_void_p * len(shards))(*[sh._h for sh in shards])
    check(lib().cupso_shard_p2p(arr, len(shards)))


def init_shards(shards: list["Swarm"]) -> None:
    """(Re)initialise host-exchanged shards: local init_swarm, then every shard
    adopts the swarm-wide initial gbest."""
    for sh in shards:
        sh.init()
    recs = [sh.snapshot_record() for sh in shards]
    for sh in shards:
        sh.adopt(recs)


def step_shards(shards: list["Swarm"], iters: int = 1) -> None:
    """cuda-sync over host-exchanged shards: propose, exchange, commit per iteration."""
    for _ in range(iters):
        recs = [sh.propose() for sh in shards]
        for sh in shards:
            sh.commit(recs)


def decode_record(rec: bytes, dims: int):
    """(fit, particle, admitted, pos) from a shard candidate record."""
    head = np.frombuffer(rec[:16], dtype=np.uint8)
    fit = float(np.frombuffer(head[:8].tobytes(), dtype=np.float64)[0])
    particle, admitted = np.frombuffer(head[8:16].tobytes(), dtype=np.uint32)
    pos = np.frombuffer(rec[16:16 + 8 * dims], dtype=np.float64).copy()
    return fit, int(particle), int(admitted), pos


def encode_record(fit: float, particle: int, admitted: int, pos) -> bytes:
    return (np.array([fit], np.float64).tobytes() +
            np.array([particle, admitted], np.uint32).tobytes() +
            np.asarray(pos, np.float64).tobytes())


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().cupso_nccl_unique_id(buf))
    return buf.raw


def shard_range(particle_cnt: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous global range [r*N/G, (r+1)*N/G) of rank r."""
    first = particle_cnt * rank // world
    last = particle_cnt * (rank + 1) // world
    return first, last - first


def select_winner(records: list[tuple[float, int]], snap_fit: float) -> int:
    """Index of the record every shard adopts, or -1: beats() among records
    (engine.hpp:38-41), then strict > against the snapshot (engine_reduction.hpp:87)."""
    best, bf, bi = -1, float("-inf"), NO_PARTICLE
    for k, (f, i) in enumerate(records):
        if i == NO_PARTICLE:
            continue
        if f > bf or (f == bf and i < bi):
            best, bf, bi = k, f, i
    return best if best >= 0 and bf > snap_fit else -1


def spec_decide(records, t0: int, K: int, kspec: int, kmax: int, t_end: int) -> dict:
    """Host mirror of spec_decide (csrc/cupso_spec.cuh): the decision every rank
    takes after a speculative pass over [t0, t0+K) from the all-gathered shard
    records (tmin, admitted, fit, particle). Returns the winner's record index
    (-1: none), whether the pass failed, and the next pass's (t0, K, kspec)."""
    tl = t0 + K - 1
    tm = min(r[0] for r in records)
    if tm < tl:  # an admission before the last iteration: re-run [t0, tm] exactly
        return dict(failed=True, winner=-1, t0=t0, K=tm - t0 + 1, kspec=max(1, kspec // 2),
                    admitted=0)
    w, bf, bi = -1, -np.inf, NO_PARTICLE
    for k, (_, _, f, i) in enumerate(records):
        if i != NO_PARTICLE and (f > bf or (f == bf and i < bi)):
            w, bf, bi = k, f, i
    ks = min(2 * kspec, kmax) if K >= kspec else kspec
    tn = t0 + K
    return dict(failed=False, winner=w, t0=tn, K=min(ks, t_end - tn) if tn < t_end else 0, kspec=ks,
                admitted=sum(r[1] for r in records))
