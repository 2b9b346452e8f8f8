"""Tensor-parallel MLP forward across GPUs: column-parallel GEMM, then the
row-parallel GEMM fused with the all-reduce of its partial sums.

The reference evaluates ``Z = sum_r GeLU(X A_r) B_r`` in ascending rank order
inside one process (``mlp_forward_tp``, tpnumerics.py:177-185).  Here each TP
rank is one process on its own GPU holding only its (uneven, shardmap.py:
160-165) slice of A and B, and the sum over ranks is an all-reduce across
GPUs.  Mode "push" (default) does that all-reduce inside the second GEMM:

1. ``H_r, Y_r = X A_r, GeLU(X A_r)`` -- tcgen05 GEMM with the fused GeLU
   epilogue (linear.MlpShard.activations).
2. ``P_r = Y_r B_r`` -- tcgen05 GEMM whose epilogue stores every 32x32 fp32
   output box twice from the same shared-memory staging: into this rank's
   ``Z`` and, when the box's rows belong to another rank's row block, straight
   into that owner's staging slot ``r`` over NVLink (one TMA tensor store per
   box; ``ntp_gemm_bf16_red`` mode 2).  The reduce-scatter is therefore done
   tile by tile while the GEMM runs: no separate send.
3. Once every rank has pushed (device signals, no host sync), the owner of
   row block ``j`` sums slots 0..n-1 **in ascending rank order** (fp32, the
   reference's summation order) and writes the sum straight into the ``j``
   rows of every rank's ``Z``: its own and, over NVLink, the peers'
   (``ntp_reduce_into`` with n destinations).  ``Z`` ends bit-identical on
   every rank after one more handshake; there is no separate gather.

Mode "nccl" is the library baseline: the same two GEMMs with a plain local
output, then ``torch.distributed.all_reduce`` (NCCL) of ``Z``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dist import DeviceOps, _wrap
from .linear import MlpShard, mm, mm_red
from .plans import dtype_code

_READY, _PUSHED, _REDUCED = 0, 1, 2
_WORDS = 64                      # per region: one u64 per writer rank
_SIG_BYTES = 3 * _WORDS * 8


class TpMlpForward:
    """One process's TP rank of a row-parallel MLP forward over ``group``
    (default: the world).  ``cols_per_rank[r]`` are rank r's ffn columns
    (e.g. ``assignment_from_comp(smap)`` for the healthy TP-n1 replica, or
    ``assignment_from_sync(smap)`` for the degraded TP-n2 one)."""

    def __init__(self, A: np.ndarray, B: np.ndarray, cols_per_rank, tokens: int, device: int,
                 group=None, mode: str = "push", out_dtype: torch.dtype = torch.float32):
        """out_dtype: the partial sums' and Z's type -- float32 (default; the
        reference sums in fp64) or bfloat16 (half the all-reduce bytes, as
        Megatron-style TP does; the owner still accumulates in fp32)."""
        if mode not in ("push", "nccl"):
            raise ValueError(f"mode must be 'push' or 'nccl', got {mode!r}")
        if out_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("out_dtype must be torch.float32 or torch.bfloat16")
        self.out_dtype = out_dtype
        eb = 4 if out_dtype == torch.float32 else 2
        self.group, self.mode, self.device = group, mode, device
        self.rank = dist.get_rank(group)
        self.n = dist.get_world_size(group)
        if len(cols_per_rank) != self.n:
            raise ValueError(f"{len(cols_per_rank)} column shards for a TP group of {self.n}")
        if self.n > _WORDS:
            raise ValueError(f"signal page holds {_WORDS} ranks")
        self.h = int(A.shape[0])
        if self.h % 32:
            raise ValueError("hidden must be a multiple of 32")
        self.T = int(tokens)
        self.shard = MlpShard(A, B, cols_per_rank[self.rank], device=f"cuda:{device}")
        # row blocks of Z: rank j owns rows [j*Tb, min(T, (j+1)*Tb)), Tb a multiple of 32
        self.Tb = ((self.T + self.n - 1) // self.n + 31) // 32 * 32
        self.blocks = [(min(self.T, j * self.Tb), min(self.T, (j + 1) * self.Tb))
                       for j in range(self.n)]
        self.ops = DeviceOps(device)
        zb = self.T * self.h * eb
        self._z = self.ops.alloc(zb)
        self.Z = _wrap(self._z, self.T * self.h, out_dtype, device).view(self.T, self.h)
        self.epoch = 0
        if mode == "nccl":
            return
        self._stg = self.ops.alloc(self.n * self.Tb * self.h * eb)
        self._sig = self.ops.alloc(_SIG_BYTES)
        mine = {"z": self.ops.handle(self._z), "stg": self.ops.handle(self._stg),
                "sig": self.ops.handle(self._sig)}
        table = [None] * self.n
        dist.all_gather_object(table, mine, group=group)
        self.peers = [j for j in range(self.n) if j != self.rank]
        self.peer_z = {j: self.ops.open(table[j]["z"]) for j in self.peers}
        self.peer_stg = {j: self.ops.open(table[j]["stg"]) for j in self.peers}
        self.peer_sig = {j: self.ops.open(table[j]["sig"]) for j in self.peers}
        # push GEMM row map: rows of another rank's block go to that owner's slot `rank`
        rows = np.arange(self.T)
        owner = np.minimum(rows // self.Tb, self.n - 1)
        red_buf = np.where(owner == self.rank, -1, owner).astype(np.int32)
        red_row = (rows - owner * self.Tb).astype(np.int32)
        dev = f"cuda:{device}"
        self.red_buf = torch.from_numpy(red_buf).to(dev)
        self.red_row = torch.from_numpy(red_row).to(dev)
        slot = self.rank * self.Tb * self.h * eb
        self.red_bases = [(self.peer_stg[j] + slot) if j != self.rank else (self._stg + slot)
                          for j in range(self.n)]
        # owner reduce: slot r of the own staging, except slot `rank` = own Z rows;
        # the sum goes to the own block's rows of every rank's Z (own first)
        lo, hi = self.blocks[self.rank]
        self._own_rows = (lo, hi)
        srcs = [self._z + lo * self.h * eb if r == self.rank
                else self._stg + r * self.Tb * self.h * eb for r in range(self.n)]
        self._srcs = _lib.ptr_array(srcs)
        dsts = [self._z + lo * self.h * eb] + [self.peer_z[j] + lo * self.h * eb for j in self.peers]
        self._dsts = _lib.ptr_array(dsts)
        # signal words: region g, writer w -> page + 8*(g*_WORDS + w)
        self._post = {g: _lib.u64_ptr_array([self.peer_sig[j] + 8 * (g * _WORDS + self.rank)
                                             for j in self.peers]) for g in range(3)}
        self._wait = {g: _lib.u64_ptr_array([self._sig + 8 * (g * _WORDS + j) for j in self.peers])
                      for g in range(3)}
        self._status = torch.zeros(1, dtype=torch.int32, device=dev)

    # ------------------------------------------------------------------------

    def _signal(self, region: int, kind: str, s, spin_ns: int = 20_000_000_000) -> None:
        if not self.peers:
            return
        L = _lib.load()
        sp = ctypes.c_void_p(s.cuda_stream)
        if kind == "post":
            _lib.check(L.ntp_signal_post(self._post[region], len(self.peers), self.epoch, sp),
                       "ntp_signal_post")
        else:
            st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
            _lib.check(L.ntp_signal_wait(self._wait[region], len(self.peers), self.epoch, spin_ns,
                                         st, sp), "ntp_signal_wait")

    def forward(self, X: torch.Tensor, stream=None) -> torch.Tensor:
        """Z = sum_r GeLU(X A_r) B_r (fp32 [T, h], identical on every rank) for
        bf16 X [T, h] (the same X on every rank).  Stream-ordered on `stream`.
        The returned tensor is this rank's (IPC-shared) output buffer: the next
        forward overwrites it, so consume or copy it first."""
        if tuple(X.shape) != (self.T, self.h) or X.dtype != torch.bfloat16:
            raise ValueError(f"X must be bf16 [{self.T}, {self.h}]")
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        sh = self.shard
        with torch.cuda.stream(s):
            if self.mode == "nccl":
                sh.activations(X)
                mm(sh.Y[:, :sh.n], sh.W[:, 1, :].T, self.Z, stream=s)
                dist.all_reduce(self.Z, group=self.group)
                return self.Z
            self.epoch += 1
            # 1. this rank's staging slots and Z are free (its previous forward is done)
            self._signal(_READY, "post", s)
            sh.activations(X)
            # 2. every owner's staging is free before this GEMM pushes into it
            self._signal(_READY, "wait", s)
            mm_red(sh.Y[:, :sh.n], sh.W[:, 1, :].T, self.Z, 1.0, self.red_buf, self.red_row,
                   self.red_bases, self.h, stream=s, mode="push_tma")
            self._signal(_PUSHED, "post", s)
            self._signal(_PUSHED, "wait", s)
            # 3. own row block: slots 0..n-1 summed in rank order (slot rank = own Z
            # rows), written into this block of every rank's Z (peer stores over NVLink)
            lo, hi = self._own_rows
            if hi > lo:
                _lib.check(_lib.load().ntp_reduce_into(
                    self._srcs, self.n, (hi - lo) * self.h, dtype_code(self.out_dtype),
                    self._dsts, self.n, ctypes.c_void_p(s.cuda_stream)), "ntp_reduce_into")
            # 4. every block has landed in this rank's Z
            self._signal(_REDUCED, "post", s)
            self._signal(_REDUCED, "wait", s)
        return self.Z

    def status(self) -> int:
        return int(self._status.item()) if self.mode == "push" else 0

    def close(self) -> None:
        """Collective: unmap the peers' buffers, then free this rank's."""
        torch.cuda.synchronize(self.device)
        if self.mode == "push":
            for d in (self.peer_z, self.peer_stg, self.peer_sig):
                for p in d.values():
                    self.ops.close(p)
        dist.barrier(group=self.group)
        self.ops.free(self._z)
        if self.mode == "push":
            self.ops.free(self._stg)
            self.ops.free(self._sig)
