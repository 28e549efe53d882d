"""Host-side mirror of the reference's psokit solver API over libcupso.so.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/psokit), so code written against psokit reads
the same here:

    pso_params / make_params          params.hpp:14-66
    fitness_fn / find_fitness         fitness.hpp:28-43, 87-103
    rng_key                           rng.hpp:10-12
    run_result                        engine.hpp:16-26
    engine_entry / engine_registry /
    find_engine                       engines.hpp:12-48
    exec_options                      group_runtime.hpp:217-222 (device knob added)

Every engine here runs on the GPU through the C-ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import check, lib

NO_PARTICLE = 0xFFFFFFFF
FIT_SENTINEL = float("-inf")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


# ------------------------------------------------------------------ params
@dataclass
class pso_params:
    """psokit::pso_params (params.hpp:14-25)."""
    inertia: float = 1.0
    cognitive: float = 2.0
    social: float = 2.0
    min_pos: float = -100.0
    max_pos: float = 100.0
    min_v: float = -100.0
    max_v: float = 100.0
    particle_cnt: int = 0
    dims: int = 1
    max_iter: int = 1
    group_size: int = 128

    def group_count(self) -> int:
        return (self.particle_cnt + self.group_size - 1) // self.group_size

    def lane_count(self) -> int:
        return self.group_count() * self.group_size

    def to_c(self) -> _lib.cupso_params:
        return _lib.cupso_params(self.inertia, self.cognitive, self.social, self.min_pos,
                                 self.max_pos, self.min_v, self.max_v, self.particle_cnt,
                                 self.dims, self.max_iter, self.group_size)

    def validate(self) -> None:
        """Raises ValueError (std::invalid_argument) naming the violated bound."""
        for name in ("particle_cnt", "dims", "max_iter", "group_size"):
            v = getattr(self, name)
            if not (0 <= v <= 0xFFFFFFFF):
                raise ValueError(f"pso_params: {name} out of uint32 range")
        p = self.to_c()
        check(lib().cupso_validate_params(C.byref(p)))


# ----------------------------------------------------------------- fitness
@dataclass(frozen=True)
class fitness_fn:
    """psokit::fitness_fn (fitness.hpp:28-43), identified by name on device."""
    name: str
    lo: float
    hi: float
    id: int

    def eval(self, x, device: int = 0) -> float:
        """Unchecked evaluation of one point, on the GPU."""
        return float(self.eval_batch(np.asarray(x, dtype=np.float64).reshape(-1, 1), device)[0])

    def eval_batch(self, x_axis_major: np.ndarray, device: int = 0) -> np.ndarray:
        """Evaluate n points given as a (dims, n) axis-major array, on the GPU."""
        x = np.ascontiguousarray(x_axis_major, dtype=np.float64)
        if x.ndim == 1:
            x = x.reshape(-1, 1)
        d, n = x.shape
        out = np.empty(n)
        check(lib().cupso_eval_fitness(device, self.id, _dp(x), n, d, _dp(out)))
        return out

    def __call__(self, x, device: int = 0) -> float:
        """Checked evaluation (fitness.hpp:35-42): DomainError outside [lo, hi]."""
        x = np.asarray(x, dtype=np.float64).reshape(-1)
        for i, v in enumerate(x):
            if not (self.lo <= v <= self.hi):
                raise _lib.DomainError(
                    f"{self.name}: component {i} outside [{self.lo:f}, {self.hi:f}]")
        return self.eval(x, device)


def fitness_registry() -> list[fitness_fn]:
    """fitness.hpp:87-95 plus the harness Rastrigin."""
    out = []
    i = 0
    while True:
        name = lib().cupso_fitness_name(i)
        if not name:
            break
        lo, hi = C.c_double(), C.c_double()
        check(lib().cupso_fitness_box(i, C.byref(lo), C.byref(hi)))
        out.append(fitness_fn(name.decode(), lo.value, hi.value, i))
        i += 1
    return out


def find_fitness(name: str) -> fitness_fn:
    """fitness.hpp:97-103: ValueError listing the known names when unknown."""
    fid = lib().cupso_fitness_id(name.encode())
    if fid < 0:
        raise ValueError(lib().cupso_last_error().decode())
    return fitness_registry()[fid]


def make_params(f: fitness_fn, particle_cnt: int, dims: int, max_iter: int,
                group_size: int = 128) -> pso_params:
    """params.hpp:52-66: box from the fitness, max_v = (hi - lo) / 2."""
    p = pso_params(min_pos=f.lo, max_pos=f.hi, max_v=(f.hi - f.lo) / 2.0,
                   min_v=-((f.hi - f.lo) / 2.0), particle_cnt=particle_cnt, dims=dims,
                   max_iter=max_iter, group_size=group_size)
    p.validate()
    return p


@dataclass(frozen=True)
class rng_key:
    """rng.hpp:10-12."""
    seed: int = 0


@dataclass
class exec_options:
    """group_runtime.hpp:217-222. threads / jitter have no GPU meaning and are
    accepted for signature compatibility; `device` selects the GPU. `devices`
    (the device-list knob SURVEY 8(b) asks for): shard one cuda-sync swarm over
    these GPUs in this process -- contiguous global particle ranges, the pass
    records exchanged over peer memory inside the pass kernel -- with a
    trajectory bit-identical to the single-GPU run."""
    threads: int = 0
    contexts_per_group: int = 0
    schedule_jitter: Optional[Callable] = None
    device: int = 0
    devices: Optional[tuple] = None


# ----------------------------------------------------------------- results
@dataclass
class swarm_state:
    """psokit::swarm_state (swarm.hpp:28-43) as numpy arrays (axis-major)."""
    particle_cnt: int
    dims: int
    positions: np.ndarray
    velocities: np.ndarray
    fitness: np.ndarray
    pbest_pos: np.ndarray
    pbest_fit: np.ndarray

    def particle_position(self, i: int) -> np.ndarray:
        return self.positions[i::self.particle_cnt][: self.dims]


@dataclass
class global_best:
    """psokit::global_best (swarm.hpp:49-54), lock word omitted."""
    fit: float
    pos: np.ndarray
    particle: int


@dataclass
class run_result:
    """psokit::run_result (engine.hpp:16-26) + the per-iteration gbest index."""
    gbest_fit: float = FIT_SENTINEL
    gbest_pos: np.ndarray = field(default_factory=lambda: np.zeros(0))
    gbest_particle: int = NO_PARTICLE
    initial_gbest_fit: float = FIT_SENTINEL
    trace: np.ndarray = field(default_factory=lambda: np.zeros(0))
    compute_seconds: float = 0.0
    queue_occupancy: np.ndarray = field(default_factory=lambda: np.zeros(0))
    trace_particle: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


iteration_observer = Callable[[int, swarm_state, global_best], None]


def run_cuda(p: pso_params, f: fitness_fn, key: rng_key, variant: int,
             opts: Optional[exec_options] = None,
             observe: Optional[iteration_observer] = None) -> run_result:
    """The engine_fn body: one full run on the GPU through cupso_run."""
    opts = opts or exec_options()
    p.validate()
    if opts.devices is not None and len(opts.devices) > 1:
        return run_sharded(p, f, key, variant, tuple(int(x) for x in opts.devices), observe)
    cp = p.to_c()
    T, d = p.max_iter, p.dims
    gpos = np.zeros(d)
    trace = np.zeros(T)
    tp = np.zeros(T, dtype=np.uint32)
    occ = np.zeros(T)
    res = _lib.cupso_result(0.0, 0, 0.0, 0.0, _dp(gpos), _dp(trace), _up(tp), _dp(occ), 0)
    err: list[BaseException] = []
    if observe is not None:
        def cb(it, view_p, _user):
            if err:
                return
            try:
                v = view_p.contents
                n, dd = v.particle_cnt, v.dims
                cells = n * dd
                s = swarm_state(
                    n, dd,
                    np.ctypeslib.as_array(v.positions, (cells,)).copy(),
                    np.ctypeslib.as_array(v.velocities, (cells,)).copy(),
                    np.ctypeslib.as_array(v.fitness, (n,)).copy(),
                    np.ctypeslib.as_array(v.pbest_pos, (cells,)).copy(),
                    np.ctypeslib.as_array(v.pbest_fit, (n,)).copy())
                gb = global_best(v.gbest_fit, np.ctypeslib.as_array(v.gbest_pos, (dd,)).copy(),
                                 v.gbest_particle)
                observe(it, s, gb)
            except BaseException as e:  # re-raised after the C call returns
                err.append(e)
        cfn = _lib.OBSERVER_FN(cb)
    else:
        cfn = _lib.OBSERVER_FN()
    st = lib().cupso_run(C.byref(cp), f.id, key.seed & 0xFFFFFFFFFFFFFFFF, variant, opts.device,
                         cfn, None, C.byref(res))
    if err:
        raise err[0]
    check(st)
    return run_result(res.gbest_fit, gpos, res.gbest_particle, res.initial_gbest_fit, trace,
                      res.compute_seconds, occ if res.has_occupancy else np.zeros(0), tp)


def run_sharded(p: pso_params, f: fitness_fn, key: rng_key, variant: int, devices: tuple,
                observe: Optional[iteration_observer] = None) -> run_result:
    """cuda-sync with the swarm sharded over several GPUs of this process
    (exec_options.devices): shard r holds the global range shard_range(N, G, r)
    on devices[r]; init_swarm per shard plus the swarm-wide initial gbest; the
    speculative passes exchange their records over peer memory (one thread per
    shard), or -- for shapes without a pass kernel -- every iteration's
    candidates through the host. compute_seconds = the slowest shard's device
    time of the iteration loop (fused exchange), or the wall time of the
    host-exchanged loop."""
    import threading
    import time

    from .swarm import Swarm, init_shards, p2p_shards, shard_range, step_shards
    if variant != _lib.SYNC:
        raise ValueError("exec_options.devices: only cuda-sync shards one swarm over several GPUs")
    if observe is not None:
        raise ValueError("exec_options.devices: the per-iteration observer needs a single-device run")
    G, T = len(devices), p.max_iter
    parts = []
    try:
        for r in range(G):
            a, c = shard_range(p.particle_cnt, G, r)
            parts.append(Swarm(p, f, key, device=devices[r], first=a, count=c, init=False))
        init_shards(parts)
        try:
            p2p_shards(parts)
            fused = True
        except ValueError:  # no speculative kernel for this shape
            fused = False
        secs = [0.0] * G
        if fused:
            errs: list[BaseException] = []

            def go(r):
                try:
                    secs[r] = parts[r].step(variant, T)
                except BaseException as e:  # re-raised below
                    errs.append(e)
            ths = [threading.Thread(target=go, args=(r,)) for r in range(G)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            if errs:
                raise errs[0]
        else:
            for sh in parts:
                sh.synchronize()
            t0 = time.perf_counter()
            step_shards(parts, T)
            for sh in parts:
                sh.synchronize()
            secs = [time.perf_counter() - t0]
        tr, tp, occ = parts[0].trace()
        gb = parts[0].gbest()
        init_fit, _ = parts[0].initial_gbest()
        return run_result(gb.fit, gb.pos, gb.particle, init_fit, tr, max(secs), occ, tp)
    finally:
        for sh in parts:
            sh.close()


# ----------------------------------------------------------------- engines
@dataclass(frozen=True)
class engine_entry:
    """psokit::engine_entry (engines.hpp:15-19). `deterministic` marks the
    engines whose trace is bitwise equal to serial (all but cuda-async)."""
    name: str
    parallel: bool
    run: Callable[..., run_result]
    deterministic: bool = True
    variant: int = -1


def _make_entry(v: int) -> engine_entry:
    name = lib().cupso_variant_name(v).decode()

    def run(p, f, key, opts=None, observe=None, _v=v):
        return run_cuda(p, f, key if isinstance(key, rng_key) else rng_key(int(key)), _v, opts, observe)

    # parallel means "bitwise equal to run_serial" in the reference's acceptance
    # (acceptance.cpp:57-59), as in the C++ adapter: not cuda-async / cuda-sync-f32
    det = bool(lib().cupso_variant_deterministic(v))
    return engine_entry(name, det, run, det, v)


def engine_registry() -> list[engine_entry]:
    """engines.hpp:21-40 with the CUDA engines."""
    return [_make_entry(v) for v in range(lib().cupso_variant_count())]


def find_engine(name: str) -> engine_entry:
    """engines.hpp:42-48: ValueError listing the known names when unknown."""
    v = lib().cupso_variant_id(name.encode())
    if v < 0:
        raise ValueError(lib().cupso_last_error().decode())
    return _make_entry(v)


def device_count() -> int:
    return lib().cupso_device_count()
