"""ctypes binding of libcupso.so (the C-ABI declared in include/cupso.h).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises. Build it with ``python -m paper_2205_01313_b200.build``
(or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CUPSO_LIB") or os.path.join(PKG_DIR, "libcupso.so")

CUPSO_OK, CUPSO_EINVAL, CUPSO_ERUNTIME, CUPSO_ELOGIC, CUPSO_EDOMAIN, CUPSO_ECUDA = range(6)
REDUCTION, UNROLLED, QUEUE, QUEUE_LOCK, SYNC, ASYNC, SYNC_F32 = range(7)


class cupso_params(C.Structure):
    _fields_ = [
        ("inertia", C.c_double), ("cognitive", C.c_double), ("social", C.c_double),
        ("min_pos", C.c_double), ("max_pos", C.c_double),
        ("min_v", C.c_double), ("max_v", C.c_double),
        ("particle_cnt", C.c_uint32), ("dims", C.c_uint32),
        ("max_iter", C.c_uint32), ("group_size", C.c_uint32),
    ]


class cupso_state_view(C.Structure):
    _fields_ = [
        ("particle_cnt", C.c_uint32), ("dims", C.c_uint32),
        ("positions", C.POINTER(C.c_double)), ("velocities", C.POINTER(C.c_double)),
        ("fitness", C.POINTER(C.c_double)), ("pbest_pos", C.POINTER(C.c_double)),
        ("pbest_fit", C.POINTER(C.c_double)),
        ("gbest_fit", C.c_double), ("gbest_particle", C.c_uint32),
        ("gbest_pos", C.POINTER(C.c_double)),
    ]


OBSERVER_FN = C.CFUNCTYPE(None, C.c_uint32, C.POINTER(cupso_state_view), C.c_void_p)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class cupso_result(C.Structure):
    _fields_ = [
        ("gbest_fit", C.c_double), ("gbest_particle", C.c_uint32),
        ("initial_gbest_fit", C.c_double), ("compute_seconds", C.c_double),
        ("gbest_pos", C.POINTER(C.c_double)), ("trace", C.POINTER(C.c_double)),
        ("trace_particle", C.POINTER(C.c_uint32)), ("queue_occupancy", C.POINTER(C.c_double)),
        ("has_occupancy", C.c_uint32),
    ]


_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_uint32)
_vp = C.c_void_p

# name -> (restype, argtypes); every function include/cupso.h declares
SIGNATURES = {
    "cupso_abi_version": (C.c_int, []),
    "cupso_last_error": (C.c_char_p, []),
    "cupso_fitness_id": (C.c_int, [C.c_char_p]),
    "cupso_fitness_name": (C.c_char_p, [C.c_int]),
    "cupso_fitness_box": (C.c_int, [C.c_int, _dp, _dp]),
    "cupso_variant_id": (C.c_int, [C.c_char_p]),
    "cupso_variant_name": (C.c_char_p, [C.c_int]),
    "cupso_variant_count": (C.c_int, []),
    "cupso_variant_deterministic": (C.c_int, [C.c_int]),
    "cupso_validate_params": (C.c_int, [C.POINTER(cupso_params)]),
    "cupso_make_params": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(cupso_params)]),
    "cupso_device_count": (C.c_int, []),
    "cupso_run": (C.c_int, [C.POINTER(cupso_params), C.c_int, C.c_uint64, C.c_int, C.c_int,
                            OBSERVER_FN, _vp, C.POINTER(cupso_result)]),
    "cupso_create": (C.c_int, [C.POINTER(cupso_params), C.c_int, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    "cupso_create_shard": (C.c_int, [C.POINTER(cupso_params), C.c_int, C.c_uint64, C.c_int,
                                     C.c_uint32, C.c_uint32, C.POINTER(_vp)]),
    "cupso_destroy": (C.c_int, [_vp]),
    "cupso_init": (C.c_int, [_vp]),
    "cupso_step": (C.c_int, [_vp, C.c_int, C.c_uint32, _dp]),
    "cupso_synchronize": (C.c_int, [_vp]),
    "cupso_iteration": (C.c_uint32, [_vp]),
    "cupso_get_gbest": (C.c_int, [_vp, _dp, _up, _dp]),
    "cupso_get_initial_gbest": (C.c_int, [_vp, _dp, _up]),
    "cupso_get_trace": (C.c_int, [_vp, C.c_uint32, C.c_uint32, _dp, _up, _dp]),
    "cupso_download_state": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp]),
    "cupso_upload_state": (C.c_int, [_vp, C.c_uint32, _dp, _dp, _dp, _dp, C.c_double, C.c_uint32, _dp]),
    "cupso_device_state": (C.c_int, [_vp, C.POINTER(_dp), C.POINTER(_dp), C.POINTER(_dp),
                                     C.POINTER(_dp), C.POINTER(C.c_uint64)]),
    "cupso_device_bytes": (C.c_size_t, [_vp]),
    "cupso_sync_grid_blocks": (C.c_int, [_vp]),
    "cupso_sync_mode": (C.c_int, [_vp]),
    "cupso_spec_stats": (C.c_int, [_vp, _vp, _vp, _vp]),
    "cupso_step_exchange": (C.c_int, [_vp, C.c_uint32, C.c_uint32, EXCHANGE_FN, _vp, _dp]),
    "cupso_shard_link": (C.c_int, [_vp, C.c_uint32]),
    "cupso_shard_p2p": (C.c_int, [_vp, C.c_uint32]),
    "cupso_ipc_handles": (C.c_int, [_vp, C.c_uint32, C.c_int, _vp]),
    "cupso_ipc_link": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, C.c_int]),
    "cupso_async_mode": (C.c_int, [_vp]),
    "cupso_record_bytes": (C.c_size_t, [C.c_uint32]),
    "cupso_shard_snapshot": (C.c_int, [_vp, _vp]),
    "cupso_shard_adopt": (C.c_int, [_vp, _vp, C.c_uint32]),
    "cupso_shard_propose": (C.c_int, [_vp, _vp]),
    "cupso_shard_propose_device": (C.c_int, [_vp, _vp]),
    "cupso_shard_commit": (C.c_int, [_vp, _vp, C.c_uint32]),
    "cupso_shard_commit_device": (C.c_int, [_vp, _vp, C.c_uint32]),
    "cupso_nccl_init": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "cupso_nccl_unique_id": (C.c_int, [_vp]),
    "cupso_stream": (_vp, [_vp]),
    "cupso_philox_batch": (C.c_int, [C.c_int, _up, _up, _up, C.c_size_t]),
    "cupso_uniform01_batch": (C.c_int, [C.c_int, C.c_uint64, _up, _dp, C.c_size_t]),
    "cupso_selftest_append": (C.c_int, [C.c_int, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64)]),
    "cupso_selftest_lock": (C.c_int, [C.c_int, C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                      _up]),
    "cupso_eval_fitness": (C.c_int, [C.c_int, C.c_int, _dp, C.c_uint32, C.c_uint32, _dp]),
    "cupso_eval_kinematics": (C.c_int, [C.c_int, C.POINTER(cupso_params), _dp, _dp, _dp, _dp, _dp,
                                        _dp, _dp, _dp, C.c_size_t]),
}


class CupsoError(RuntimeError):
    """Base for CUDA-side failures (CUPSO_ECUDA)."""


class LogicError(RuntimeError):
    """std::logic_error analogue (CUPSO_ELOGIC)."""


class DomainError(ValueError):
    """std::domain_error analogue (CUPSO_EDOMAIN)."""


_lib = None


def lib() -> C.CDLL:
    """Load libcupso.so once; raise loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -m paper_2205_01313_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    """Map a cupso_status onto the reference's exception types."""
    if status == CUPSO_OK:
        return
    msg = lib().cupso_last_error().decode(errors="replace")
    if status == CUPSO_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == CUPSO_ELOGIC:
        raise LogicError(msg)
    if status == CUPSO_EDOMAIN:
        raise DomainError(msg)
    if status == CUPSO_ECUDA:
        raise CupsoError(msg)
    raise RuntimeError(msg)  # std::runtime_error
