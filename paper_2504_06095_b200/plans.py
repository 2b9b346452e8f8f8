"""Device copy/reduce plans: build unit tables on the host, run them on a B200.

A plan pairs every unit (MLP column = A column + B row, or attention head) of
side A with the same unit on side B.  For a gradient sync A is the healthy
replica's copy and B the reduced replica's (tpnumerics.py:342-343 operand
order); for a reconfiguration A is the source layout and B the destination.
Buffers are referenced by index into the pointer list passed at run time, so
one plan serves local buffers (1-GPU emulation) and peer-mapped buffers alike.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

TORCH_DTYPES = {torch.float32: _lib.NTP_F32, torch.bfloat16: _lib.NTP_BF16,
                torch.float16: _lib.NTP_F16, torch.float64: _lib.NTP_F64}
OPS = {"sum": _lib.NTP_OP_SUM, "mean": _lib.NTP_OP_MEAN, "weighted": _lib.NTP_OP_WEIGHTED}


def dtype_code(dtype: torch.dtype) -> int:
    try:
        return TORCH_DTYPES[dtype]
    except KeyError:
        raise ValueError(f"unsupported gradient dtype {dtype}") from None


def layout_offsets(cols_per_rank, k: int, unit: int, base=None):
    """owner[j], element offset[j] of column j in a unit-major per-rank layout.

    cols_per_rank[r] lists rank r's columns in storage order (the reference's
    per-rank ``cols``, tpnumerics.py:137); base[r] is where the segment starts
    inside rank r's buffer (elements).
    """
    owner = np.full(k, -1, dtype=np.int64)
    off = np.full(k, -1, dtype=np.int64)
    for r, cols in enumerate(cols_per_rank):
        cols = np.asarray(cols, dtype=np.int64)
        owner[cols] = r
        off[cols] = np.arange(len(cols), dtype=np.int64) * unit + (0 if base is None else int(base[r]))
    if (owner < 0).any():
        raise ValueError("assignment does not partition the columns exactly once")
    return owner, off


class Plan:
    """Owns an ``ntp_plan`` (include/ntp_b200.h)."""

    def __init__(self, dtype: int):
        self._L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._L.ntp_plan_create(ctypes.byref(h), int(dtype)), "ntp_plan_create")
        self._h = h
        self.dtype = int(dtype)
        self.device = None

    def add_units(self, unit_elems: int, a_buf, a_off, b_buf, b_off) -> "Plan":
        a_buf, b_buf = _lib.i32(a_buf), _lib.i32(b_buf)
        a_off, b_off = _lib.i64(a_off), _lib.i64(b_off)
        n = len(a_buf)
        if not (len(a_off) == len(b_buf) == len(b_off) == n):
            raise ValueError("unit arrays differ in length")
        _lib.check(self._L.ntp_plan_add_units(self._h, n, int(unit_elems), _lib.p32(a_buf),
                                              _lib.p64(a_off), _lib.p32(b_buf), _lib.p64(b_off)),
                   "ntp_plan_add_units")
        return self

    def finalize(self) -> "Plan":
        _lib.check(self._L.ntp_plan_finalize(self._h), "ntp_plan_finalize")
        return self

    def upload(self, device: int) -> "Plan":
        _lib.check(self._L.ntp_plan_upload(self._h, int(device)), "ntp_plan_upload")
        self.device = int(device)
        return self

    @property
    def stats(self) -> dict:
        s = _lib.PlanStats()
        _lib.check(self._L.ntp_plan_stats_get(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _lib.PlanStats._fields_}

    def export(self) -> np.ndarray:
        """Chunk table as int64 [n_chunks, 5] = (a_buf, a_off, b_buf, b_off, len)."""
        n = self.stats["n_chunks"]
        out = np.empty((max(n, 1), 5), dtype=np.int64)
        _lib.check(self._L.ntp_plan_export(self._h, _lib.p64(out)))
        return out[:n]

    # -- device execution ------------------------------------------------------

    def check(self, buf_elems, write_sides: int = 3) -> "Plan":
        """Static memory-safety check (ntp_plan_check): every chunk inside its
        buffer (buf_elems[b] elements) and no element written twice on the
        sides in write_sides (3: a sync, 2: a reshard copy).  ValueError names
        the offending chunk."""
        sizes = np.ascontiguousarray(buf_elems, dtype=np.int64)
        _lib.check(self._L.ntp_plan_check(self._h, _lib.p64(sizes), len(sizes), int(write_sides)),
                   "ntp_plan_check")
        return self

    def grad_sync(self, bufs, op: int, w_a: float = 1.0, w_b: float = 1.0, stream=None) -> None:
        ptrs = _lib.ptr_array(bufs)
        _lib.check(self._L.ntp_grad_sync(self._h, ptrs, len(bufs), int(op), float(w_a),
                                         float(w_b), _stream_ptr(stream, self.device)),
                   "ntp_grad_sync")

    def grad_sync_into(self, bufs, op: int, w_a: float, w_b: float, write_mask: int,
                       stream=None) -> None:
        """grad_sync writing only the sides in write_mask (1: A, 2: B, 3: both)."""
        _lib.check(self._L.ntp_grad_sync_ex(self._h, _lib.ptr_array(bufs), len(bufs), int(op),
                                            float(w_a), float(w_b), int(write_mask),
                                            _stream_ptr(stream, self.device)), "ntp_grad_sync_ex")

    def reshard(self, bufs, stream=None) -> None:
        ptrs = _lib.ptr_array(bufs)
        _lib.check(self._L.ntp_reshard(self._h, ptrs, len(bufs), _stream_ptr(stream, self.device)),
                   "ntp_reshard")

    def grad_sync_signaled(self, bufs, op, w_a, w_b, wait, post, epoch, spin_ns, status_ptr,
                           stream=None) -> None:
        _lib.check(self._L.ntp_grad_sync_signaled(
            self._h, _lib.ptr_array(bufs), len(bufs), int(op), float(w_a), float(w_b),
            _lib.u64_ptr_array(wait), len(wait), _lib.u64_ptr_array(post), len(post),
            int(epoch), int(spin_ns), ctypes.cast(int(status_ptr), ctypes.POINTER(ctypes.c_int)),
            _stream_ptr(stream, self.device)), "ntp_grad_sync_signaled")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._L.ntp_plan_destroy(h)
            except Exception:
                pass
            self._h = None


def _stream_ptr(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(int(stream.cuda_stream if hasattr(stream, "cuda_stream") else stream))


def tensor_ptrs(tensors) -> list[int]:
    return [int(t.data_ptr()) for t in tensors]


class MultiPlan:
    """Owns an ``ntp_mplan``: R-way unit tables for DP > 2 syncs."""

    def __init__(self, dtype: int, R: int):
        self._L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._L.ntp_mplan_create(ctypes.byref(h), int(dtype), int(R)), "ntp_mplan_create")
        self._h, self.dtype, self.R, self.device = h, int(dtype), int(R), None

    def add_units(self, unit_elems: int, bufs, offs) -> "MultiPlan":
        """bufs, offs: [R x n_units] arrays (replica-major)."""
        b = np.ascontiguousarray(bufs, dtype=np.int32)
        o = np.ascontiguousarray(offs, dtype=np.int64)
        if b.shape != o.shape or b.ndim != 2 or b.shape[0] != self.R:
            raise ValueError("bufs/offs must be [R x n_units]")
        _lib.check(self._L.ntp_mplan_add_units(self._h, b.shape[1], int(unit_elems), _lib.p32(b),
                                               _lib.p64(o)), "ntp_mplan_add_units")
        return self

    def finalize(self) -> "MultiPlan":
        _lib.check(self._L.ntp_mplan_finalize(self._h), "ntp_mplan_finalize")
        return self

    @property
    def n_chunks(self) -> int:
        return _lib.check(self._L.ntp_mplan_chunks(self._h))

    def upload(self, device: int) -> "MultiPlan":
        _lib.check(self._L.ntp_mplan_upload(self._h, int(device)), "ntp_mplan_upload")
        self.device = int(device)
        return self

    def sync(self, bufs, op: int, weights=None, stream=None) -> None:
        w = None
        if weights is not None:
            w = np.ascontiguousarray(weights, dtype=np.float64)
            if len(w) != self.R:
                raise ValueError("one weight per replica")
            w = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        _lib.check(self._L.ntp_multi_sync(self._h, _lib.ptr_array(bufs), len(bufs), int(op), w,
                                          _stream_ptr(stream, self.device)), "ntp_multi_sync")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._L.ntp_mplan_destroy(h)
            except Exception:
                pass
            self._h = None
