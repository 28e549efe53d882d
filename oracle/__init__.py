"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to the CPU oracle.

Two checkers live here:

* ``Oracle``   -- oracle/_build/liboracle.so, the plain-C restatement of the
                  reference serial solver (oracle/pso_oracle.c).
* ``Reference`` -- oracle/_ref/libpsokit_ref.so, the UNMODIFIED reference
                  (psokit headers from /root/reference) behind a C shim
                  (oracle/ref_shim.cpp). Only buildable where /root/reference
                  exists; the prebuilt .so travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package. The product (paper_2205_01313_b200, libcupso.so)
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpsokit_ref.so")
REF_INC = "/root/reference/proj/include"

FITNESS = ["cubic", "sphere", "rosenbrock", "griewank", "rastrigin"]


def build(ref: bool = True) -> None:
    """Build the oracle (and the reference shim when the reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_INC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class orc_params(C.Structure):
    _fields_ = [
        ("inertia", C.c_double), ("cognitive", C.c_double), ("social", C.c_double),
        ("min_pos", C.c_double), ("max_pos", C.c_double),
        ("min_v", C.c_double), ("max_v", C.c_double),
        ("particle_cnt", C.c_uint32), ("dims", C.c_uint32),
        ("max_iter", C.c_uint32), ("group_size", C.c_uint32),
    ]


class orc_state(C.Structure):
    _fields_ = [
        ("particle_cnt", C.c_uint32), ("dims", C.c_uint32),
        ("positions", C.POINTER(C.c_double)), ("velocities", C.POINTER(C.c_double)),
        ("fitness", C.POINTER(C.c_double)), ("pbest_pos", C.POINTER(C.c_double)),
        ("pbest_fit", C.POINTER(C.c_double)),
    ]


class orc_result(C.Structure):
    _fields_ = [
        ("gbest_fit", C.c_double), ("gbest_particle", C.c_uint32),
        ("initial_gbest_fit", C.c_double), ("initial_gbest_particle", C.c_uint32),
        ("gbest_pos", C.POINTER(C.c_double)), ("trace", C.POINTER(C.c_double)),
        ("trace_particle", C.POINTER(C.c_uint32)), ("compute_seconds", C.c_double),
    ]


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


@dataclass
class OracleRun:
    trace: np.ndarray
    trace_particle: np.ndarray
    gbest_pos: np.ndarray
    gbest_fit: float
    gbest_particle: int
    initial_gbest_fit: float
    compute_seconds: float
    state: dict = field(default_factory=dict)


class Oracle:
    """The C restatement (oracle/pso_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.L = L
        L.orc_uniform01.restype = C.c_double
        L.orc_uniform01.argtypes = [C.c_uint64] + [C.c_uint32] * 4
        L.orc_fitness_eval.restype = C.c_double
        L.orc_fitness_eval.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_size_t]
        L.orc_velocity_step.restype = C.c_double
        L.orc_velocity_step.argtypes = [C.c_double] * 4 + [C.POINTER(orc_params), C.c_double, C.c_double]
        L.orc_position_step.restype = C.c_double
        L.orc_position_step.argtypes = [C.c_double, C.c_double, C.POINTER(orc_params)]
        L.orc_make_params.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.POINTER(orc_params), C.c_char_p, C.c_size_t]
        L.orc_validate.argtypes = [C.POINTER(orc_params), C.c_char_p, C.c_size_t]
        L.orc_run_serial.argtypes = [C.POINTER(orc_params), C.c_int, C.c_uint64, C.POINTER(orc_result),
                                     C.POINTER(orc_state), C.c_void_p, C.c_void_p]
        L.orc_trimmed_mean.restype = C.c_double
        L.orc_trimmed_mean.argtypes = [C.POINTER(C.c_double), C.c_size_t]
        L.orc_trace_checksum.argtypes = [C.POINTER(C.c_double), C.c_size_t, C.c_char_p]
        L.orc_shard_step.argtypes = [C.POINTER(orc_params), C.c_int, C.c_uint64, C.c_uint32, C.POINTER(orc_state),
                                     C.c_uint32, C.c_uint32, C.POINTER(C.c_double), C.c_double,
                                     C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                     C.POINTER(C.c_uint32)]
        L.orc_init_swarm.argtypes = [C.POINTER(orc_params), C.c_uint64, C.c_int, C.POINTER(orc_state),
                                     C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_double)]

    # -- primitives ---------------------------------------------------------
    def philox(self, ctr, k0, k1):
        c = (C.c_uint32 * 4)(*ctr)
        o = (C.c_uint32 * 4)()
        self.L.orc_philox4x32(c, C.c_uint32(k0), C.c_uint32(k1), o)
        return tuple(o)

    def uniform01(self, seed, it, particle, axis, slot):
        return self.L.orc_uniform01(seed, it, particle, axis, slot)

    def fitness(self, name, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.L.orc_fitness_eval(FITNESS.index(name), _dp(x), x.size, 1)

    def make_params(self, fitness, particles, dims, iters, group_size=128):
        p = orc_params()
        msg = C.create_string_buffer(256)
        rc = self.L.orc_make_params(FITNESS.index(fitness), particles, dims, iters, group_size,
                                    C.byref(p), msg, 256)
        if rc != 0:
            raise ValueError(msg.value.decode())
        return p

    def velocity_step(self, v, x, pb, g, p, r1, r2):
        return self.L.orc_velocity_step(v, x, pb, g, C.byref(p), r1, r2)

    def position_step(self, x, v, p):
        return self.L.orc_position_step(x, v, C.byref(p))

    def checksum(self, trace):
        t = np.ascontiguousarray(trace, dtype=np.float64)
        out = C.create_string_buffer(17)
        self.L.orc_trace_checksum(_dp(t), t.size, out)
        return out.value.decode()

    def trimmed_mean(self, xs):
        a = np.ascontiguousarray(xs, dtype=np.float64)
        return self.L.orc_trimmed_mean(_dp(a), a.size)

    def init(self, fitness, particles, dims, seed):
        p = self.make_params(fitness, particles, dims, 1)
        cells = particles * dims
        st = {k: np.zeros(cells) for k in ("positions", "velocities", "pbest_pos")}
        st.update({k: np.zeros(particles) for k in ("fitness", "pbest_fit")})
        s = orc_state(particles, dims, _dp(st["positions"]), _dp(st["velocities"]),
                      _dp(st["fitness"]), _dp(st["pbest_pos"]), _dp(st["pbest_fit"]))
        gf = C.c_double()
        gi = C.c_uint32()
        gp = np.zeros(dims)
        self.L.orc_init_swarm(C.byref(p), seed, FITNESS.index(fitness), C.byref(s), C.byref(gf),
                              C.byref(gi), _dp(gp))
        return st, gf.value, gi.value, gp

    def shard_step(self, fitness, params, seed, t, st, first, count, snap_pos, snap_fit):
        """One iteration over [first, first+count) of the full state dict `st` (in place)."""
        n, d = params.particle_cnt, params.dims
        s = orc_state(n, d, _dp(st["positions"]), _dp(st["velocities"]), _dp(st["fitness"]),
                      _dp(st["pbest_pos"]), _dp(st["pbest_fit"]))
        bf, bi, adm = C.c_double(), C.c_uint32(), C.c_uint32()
        bp = np.zeros(d)
        sp = np.ascontiguousarray(snap_pos, dtype=np.float64)
        self.L.orc_shard_step(C.byref(params), FITNESS.index(fitness), seed, t, C.byref(s), first, count,
                              _dp(sp), snap_fit, C.byref(bf), C.byref(bi), _dp(bp), C.byref(adm))
        return bf.value, bi.value, bp, adm.value

    def run_serial(self, fitness, particles, dims, iters, seed, params=None, want_state=True):
        p = params if params is not None else self.make_params(fitness, particles, dims, iters)
        n, d, T = p.particle_cnt, p.dims, p.max_iter
        trace = np.zeros(T)
        tp = np.zeros(T, dtype=np.uint32)
        gp = np.zeros(d)
        r = orc_result(0.0, 0, 0.0, 0, _dp(gp), _dp(trace), _up(tp), 0.0)
        st = {}
        sp = None
        if want_state:
            cells = n * d
            st = {k: np.zeros(cells) for k in ("positions", "velocities", "pbest_pos")}
            st.update({k: np.zeros(n) for k in ("fitness", "pbest_fit")})
            s = orc_state(n, d, _dp(st["positions"]), _dp(st["velocities"]), _dp(st["fitness"]),
                          _dp(st["pbest_pos"]), _dp(st["pbest_fit"]))
            sp = C.byref(s)
        rc = self.L.orc_run_serial(C.byref(p), FITNESS.index(fitness), seed, C.byref(r), sp, None, None)
        if rc != 0:
            raise ValueError(f"orc_run_serial failed rc={rc}")
        return OracleRun(trace, tp, gp, r.gbest_fit, r.gbest_particle, r.initial_gbest_fit,
                         r.compute_seconds, st)


class Reference:
    """The unmodified reference solver behind oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (built only where /root/reference exists)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_uniform01.restype = C.c_double
        L.ref_uniform01.argtypes = [C.c_uint64] + [C.c_uint32] * 4
        L.ref_fitness_eval.restype = C.c_double
        L.ref_fitness_eval.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_size_t]
        dp = C.POINTER(C.c_double)
        up = C.POINTER(C.c_uint32)
        L.ref_run.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                              C.c_uint64, C.c_uint32, dp, up, dp, dp, dp, up, dp, dp,
                              dp, dp, dp, dp, dp]
        L.ref_init.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64, dp, dp, dp, dp, up, dp]
        L.ref_trace_checksum.argtypes = [dp, C.c_size_t, C.c_char_p]

    def philox(self, ctr, k0, k1):
        c = (C.c_uint32 * 4)(*ctr)
        o = (C.c_uint32 * 4)()
        self.L.ref_philox4x32(c, C.c_uint32(k0), C.c_uint32(k1), o)
        return tuple(o)

    def fitness(self, name, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.L.ref_fitness_eval(name.encode(), _dp(x), x.size)

    def checksum(self, trace):
        t = np.ascontiguousarray(trace, dtype=np.float64)
        out = C.create_string_buffer(17)
        self.L.ref_trace_checksum(_dp(t), t.size, out)
        return out.value.decode()

    def run(self, engine, fitness, particles, dims, iters, seed, group_size=128, threads=0,
            want_particles=True, want_state=False):
        T, n, d = iters, particles, dims
        trace = np.zeros(T)
        tp = np.zeros(T, dtype=np.uint32) if want_particles else None
        occ = np.zeros(T)
        gp = np.zeros(d)
        gf, gi, ig, cs = C.c_double(), C.c_uint32(), C.c_double(), C.c_double()
        st = {}
        if want_state:
            st = {k: np.zeros(n * d) for k in ("positions", "velocities", "pbest_pos")}
            st.update({k: np.zeros(n) for k in ("fitness", "pbest_fit")})
        nul = C.POINTER(C.c_double)()
        sargs = [(_dp(st[k]) if want_state else nul)
                 for k in ("positions", "velocities", "fitness", "pbest_pos", "pbest_fit")]
        rc = self.L.ref_run(engine.encode(), fitness.encode(), n, d, T, group_size, seed, threads,
                            _dp(trace), _up(tp) if tp is not None else C.POINTER(C.c_uint32)(),
                            _dp(occ), _dp(gp), C.byref(gf), C.byref(gi), C.byref(ig), C.byref(cs),
                            *sargs)
        if rc != 0:
            err = self.L.ref_last_error().decode()
            raise (ValueError if rc == 1 else RuntimeError)(err)
        return OracleRun(trace, tp if tp is not None else np.zeros(0, np.uint32), gp, gf.value,
                         gi.value, ig.value, cs.value, st), occ
