"""ctypes binding of libntp_b200.so (the C ABI in include/ntp_b200.h).

There is no fallback: if the library is missing or fails to load, every entry
point raises.  ``load()`` builds the library in-tree from csrc/ when it is
absent or stale and nvcc is available (the build container); on the GPU box
the prebuilt .so from the snapshot is used.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import build as _build

NTP_OK, NTP_EINVAL, NTP_ECUDA, NTP_ENOMEM, NTP_ESTATE, NTP_ETIMEOUT = 0, -1, -2, -3, -4, -5
NTP_F32, NTP_BF16, NTP_F16, NTP_F64 = 0, 1, 2, 3
NTP_OP_SUM, NTP_OP_MEAN, NTP_OP_WEIGHTED = 0, 1, 2
NTP_PRE_SYNC, NTP_POST_SYNC = 0, 1
IPC_HANDLE_BYTES = 64

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p
_vpp = ctypes.POINTER(ctypes.c_void_p)
_u64pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_uint64))


class PlanStats(ctypes.Structure):
    _fields_ = [("n_units", ctypes.c_int64), ("n_runs", ctypes.c_int64),
                ("n_chunks", ctypes.c_int64), ("elems", ctypes.c_int64),
                ("vectorized", ctypes.c_int32), ("max_buf", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("device", ctypes.c_int32)]


# name -> (restype, argtypes); mirrors include/ntp_b200.h one to one
SIGNATURES = {
    "ntp_last_error": (ctypes.c_char_p, []),
    "ntp_abi_version": (ctypes.c_int, []),
    "ntp_set_option": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64]),
    "ntp_get_option": (ctypes.c_int64, [ctypes.c_int]),
    "ntp_shard_map": (ctypes.c_int, [ctypes.c_int64] * 3 + [_i64p, _i64p]),
    "ntp_reshard_plan": (ctypes.c_int64, [_i64p, _i64p, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int, _i64p, _i64p, _i64p]),
    "ntp_apply_plan": (ctypes.c_int, [_i64p, ctypes.c_int64, _i64p, _i64p, _i64p,
                                      ctypes.c_int64]),
    "ntp_naive_overlaps": (ctypes.c_int64, [ctypes.c_int64] * 3 + [_i64p, _i64p]),
    "ntp_interval_overlaps": (ctypes.c_int64, [ctypes.c_int64] * 3 + [_i64p]),
    "ntp_head_partition": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _i64p,
                                          ctypes.POINTER(ctypes.c_double)]),
    "ntp_plan_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int]),
    "ntp_plan_add_units": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _i32p, _i64p,
                                          _i32p, _i64p]),
    "ntp_plan_finalize": (ctypes.c_int, [_vp]),
    "ntp_plan_stats_get": (ctypes.c_int, [_vp, ctypes.POINTER(PlanStats)]),
    "ntp_plan_export": (ctypes.c_int, [_vp, _i64p]),
    "ntp_plan_check": (ctypes.c_int, [_vp, _i64p, ctypes.c_int, ctypes.c_int]),
    "ntp_plan_upload": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ntp_plan_destroy": (None, [_vp]),
    "ntp_grad_sync": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_double, _vp]),
    "ntp_grad_sync_ex": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, _vp]),
    "ntp_reshard": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, _vp]),
    "ntp_uniform_sync": (ctypes.c_int, [_vpp, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                        ctypes.c_int, ctypes.POINTER(ctypes.c_double), _vp]),
    "ntp_reduce_into": (ctypes.c_int, [_vpp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, _vpp,
                                       ctypes.c_int, _vp]),
    "ntp_mplan_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, ctypes.c_int]),
    "ntp_mplan_add_units": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _i32p, _i64p]),
    "ntp_mplan_finalize": (ctypes.c_int, [_vp]),
    "ntp_mplan_chunks": (ctypes.c_int64, [_vp]),
    "ntp_mplan_upload": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ntp_mplan_destroy": (None, [_vp]),
    "ntp_multi_sync": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_double), _vp]),
    "ntp_multi_set_kernel": (ctypes.c_int, [ctypes.c_int]),
    "ntp_gemm_bf16": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int, _vp, ctypes.c_int64,
                                     ctypes.c_int, _vp, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     _vp, ctypes.c_int64, ctypes.c_float, _vp]),
    "ntp_gemm_bf16_ex": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int, _vp, ctypes.c_int64,
                                        ctypes.c_int, _vp, ctypes.c_int64, ctypes.c_int,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int, _vp, ctypes.c_int64, ctypes.c_float,
                                        ctypes.c_int, _vp]),
    "ntp_gemm_bf16_red": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int, _vp, ctypes.c_int64,
                                         ctypes.c_int, _vp, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_float, _vp, _vp, _vpp, ctypes.c_int,
                                         ctypes.c_int64, ctypes.c_int, _vp]),
    "ntp_gemm_set_pair": (ctypes.c_int, [ctypes.c_int]),
    "ntp_gemm_set_max_ctas": (ctypes.c_int, [ctypes.c_int]),
    "ntp_gemm_get_max_ctas": (ctypes.c_int, []),
    "ntp_gemm_set_split_k": (ctypes.c_int, [ctypes.c_int]),
    "ntp_gemm_set_pdl": (ctypes.c_int, [ctypes.c_int]),
    "ntp_alloc": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, _vpp]),
    "ntp_free": (ctypes.c_int, [_vp]),
    "ntp_ipc_get_handle": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "ntp_ipc_open": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, _vpp]),
    "ntp_ipc_close": (ctypes.c_int, [_vp]),
    "ntp_grad_sync_signaled": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_double, ctypes.c_double, _u64pp,
                                              ctypes.c_int, _u64pp, ctypes.c_int,
                                              ctypes.c_uint64, ctypes.c_uint64,
                                              ctypes.POINTER(ctypes.c_int), _vp]),
    "ntp_grad_sync_step": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, _u64pp, ctypes.c_int,
                                          _u64pp, ctypes.c_int, _u64pp, ctypes.c_int, _u64pp,
                                          ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.POINTER(ctypes.c_int), _vp]),
    "ntp_signal_post": (ctypes.c_int, [_u64pp, ctypes.c_int, ctypes.c_uint64, _vp]),
    "ntp_signal_wait": (ctypes.c_int, [_u64pp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.POINTER(ctypes.c_int), _vp]),
    "ntp_grad_sync_signaled_dev": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_double, ctypes.c_double, _u64pp,
                                                  ctypes.c_int, _u64pp, ctypes.c_int, _vp,
                                                  ctypes.c_uint64, ctypes.POINTER(ctypes.c_int),
                                                  _vp]),
    "ntp_grad_sync_step_dev": (ctypes.c_int, [_vp, _vpp, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_double, ctypes.c_double, _u64pp,
                                              ctypes.c_int, _u64pp, ctypes.c_int, _u64pp,
                                              ctypes.c_int, _u64pp, ctypes.c_int, _vp,
                                              ctypes.c_uint64, ctypes.POINTER(ctypes.c_int), _vp]),
    "ntp_signal_post_dev": (ctypes.c_int, [_u64pp, ctypes.c_int, _vp, _vp]),
    "ntp_signal_wait_dev": (ctypes.c_int, [_u64pp, ctypes.c_int, _vp, ctypes.c_int,
                                           ctypes.c_uint64, ctypes.POINTER(ctypes.c_int), _vp]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load (building if needed) libntp_b200.so; raises if it cannot."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if os.environ.get("NTP_LIB_AB"):  # A/B experiments only: another build of the same ABI
            path = os.environ["NTP_LIB_AB"]
        try:
            if path == _build.LIB and _build._stale() and os.path.exists(_build.NVCC):
                _build.build()
        except Exception as e:  # pragma: no cover - surfaced below
            if not os.path.exists(path):
                raise RuntimeError(f"cannot build libntp_b200.so: {e}") from e
        if not os.path.exists(path):
            raise RuntimeError(
                f"libntp_b200.so not found at {path}; run `python -m paper_2504_06095_b200.build`"
            )
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.ntp_abi_version() != 1:
            raise RuntimeError("libntp_b200.so ABI version mismatch")
        _lib = L
        return L


def last_error() -> str:
    return load().ntp_last_error().decode()


def check(status: int, what: str = "") -> int:
    """Map a C status to the reference's exception types."""
    if status >= 0:
        return status
    msg = last_error()
    if status == NTP_EINVAL:
        raise ValueError(msg)
    if status == NTP_ETIMEOUT:
        raise TimeoutError(msg or f"{what}: cross-GPU signal timeout")
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def p64(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def p32(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


def ptr_array(ptrs) -> ctypes.Array:
    return (ctypes.c_void_p * max(len(ptrs), 1))(*[int(p) for p in ptrs])


def u64_ptr_array(ptrs):
    T = ctypes.POINTER(ctypes.c_uint64)
    return (T * max(len(ptrs), 1))(*[ctypes.cast(int(p), T) for p in ptrs])
