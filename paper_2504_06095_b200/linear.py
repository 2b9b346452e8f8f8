"""Uneven-shard column/row-parallel MLP linears on tcgen05 (``ntp_gemm_bf16``).

Per TP rank i the reference computes (tpnumerics.py:177-185, 238-252)

    H_i = X A_i        Y_i = GeLU(H_i)        Z = sum_i Y_i B_i
    dB_i = Y_i^T G     D_i = (G B_i^T) * GeLU'(H_i)     dA_i = X^T D_i

with ragged n_i columns per rank (shardmap.py:160-165).  Here every rank's
weights are stored **unit-major**, exactly like its gradients: ``W[p, 0, :]`` is
column p of A_i and ``W[p, 1, :]`` is row p of B_i.  All five GEMMs read that
layout in place (K-major or MN-major TMA views with a 2*hidden row pitch), and
the two weight-gradient GEMMs write ``grads[p, 0, :]`` / ``grads[p, 1, :]``
directly -- the arena the sync kernel consumes, with no repacking.

Numerics: bf16 operands, fp32 accumulation in TMEM; H, Y and D are kept in
bf16, Z in fp32 (the TP partial sums).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

EPI = {"none": 0, "gelu": 1, "dgelu": 2}


def _operand(t: torch.Tensor):
    """(ptr, ld, mn_major) of a logical [rows x K] bf16 view."""
    if t.dtype != torch.bfloat16:
        raise ValueError("tcgen05 GEMM operands are bf16")
    if t.dim() != 2:
        raise ValueError("GEMM operands are 2-D views")
    if t.stride(1) == 1:
        return t.data_ptr(), t.stride(0), 0
    if t.stride(0) == 1:
        return t.data_ptr(), t.stride(1), 1
    raise ValueError("GEMM operand must have a unit stride in one dimension")


PDL = {None: -1, "off": 0, "after": 1, "independent": 2}


def mm(A: torch.Tensor, Bt: torch.Tensor, out: torch.Tensor, *, epilogue: str = "none",
       aux: torch.Tensor | None = None, alpha: float = 1.0, stream=None,
       pdl: str | None = None) -> torch.Tensor:
    """out[M x N] = epilogue(A[M x K] @ Bt[N x K]^T) on the tensor cores.

    A and Bt may be K-major or MN-major views (e.g. ``Y.T``); ``out`` is a
    row-major [M x N] view with any row pitch (bf16 or fp32).
    pdl (programmatic dependent launch, ntp_gemm_bf16_ex): "after" overlaps
    the launch's set-up with the previous kernel's tail; "independent" runs it
    under that tail (the caller guarantees no data dependence either way);
    None follows ntp_gemm_set_pdl."""
    if pdl not in PDL:
        raise ValueError(f"unknown pdl mode {pdl!r}")
    M, K = A.shape
    N, K2 = Bt.shape
    if K != K2 or tuple(out.shape) != (M, N):
        raise ValueError(f"shape mismatch: A {tuple(A.shape)}, Bt {tuple(Bt.shape)}, out {tuple(out.shape)}")
    if out.stride(1) != 1:
        raise ValueError("out must be row-major")
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("out must be bf16 or fp32")
    a_ptr, lda, a_mn = _operand(A)
    b_ptr, ldb, b_mn = _operand(Bt)
    aux_ptr, ld_aux = (0, 0)
    if epilogue != "none":
        if aux is None or aux.dtype != torch.bfloat16 or tuple(aux.shape) != (M, N) or aux.stride(1) != 1:
            raise ValueError("epilogue needs a bf16 row-major aux [M x N]")
        aux_ptr, ld_aux = aux.data_ptr(), aux.stride(0)
    if stream is None:
        stream = torch.cuda.current_stream(A.device)
    L = _lib.load()
    args = (ctypes.c_void_p(a_ptr), lda, a_mn, ctypes.c_void_p(b_ptr), ldb, b_mn,
            ctypes.c_void_p(out.data_ptr()), out.stride(0), int(out.dtype == torch.float32),
            M, N, K, EPI[epilogue], ctypes.c_void_p(aux_ptr), ld_aux, float(alpha))
    sp = ctypes.c_void_p(stream.cuda_stream)
    if pdl is None:
        _lib.check(L.ntp_gemm_bf16(*args, sp), "ntp_gemm_bf16")
    else:
        _lib.check(L.ntp_gemm_bf16_ex(*args, PDL[pdl], sp), "ntp_gemm_bf16_ex")
    return out


# "red": red.add into zeroed arenas; "push": row stores into the partner's
# staging arena; "push_tma": the same, but 32-row boxes whose rows are
# consecutive in the partner's layout go as one TMA tensor store over NVLink;
# "red_tma": zeroed arenas like "red", every box added with TMA bulk tensor
# reductions (cp.reduce.async.bulk.tensor .add) -- no staging, no local tail
FUSED_MODES = {"red": 0, "push": 1, "push_tma": 2, "red_tma": 3}


def mm_red(A: torch.Tensor, Bt: torch.Tensor, out: torch.Tensor, alpha: float,
           red_buf: torch.Tensor, red_row: torch.Tensor, red_bases, red_ld: int,
           stream=None, mode: str = "red") -> None:
    """Fused wgrad + sync.  mode "red": red.add(alpha * A @ Bt^T) into ``out``
    (local copy) and into row red_row[m] of red_bases[red_buf[m]] (the partner's
    copy); both start at zero.  mode "push": plain stores into ``out`` and into
    the partner's staging arena.  red_buf/red_row: int32 device tensors [M]."""
    if mode not in FUSED_MODES:
        raise ValueError(f"unknown fused mode {mode!r}")
    M, K = A.shape
    N, K2 = Bt.shape
    if K != K2 or tuple(out.shape) != (M, N) or out.stride(1) != 1:
        raise ValueError("shape mismatch")
    if red_buf.dtype != torch.int32 or red_row.dtype != torch.int32 or len(red_buf) != M:
        raise ValueError("red_buf/red_row must be int32 [M]")
    a_ptr, lda, a_mn = _operand(A)
    b_ptr, ldb, b_mn = _operand(Bt)
    if stream is None:
        stream = torch.cuda.current_stream(A.device)
    _lib.check(_lib.load().ntp_gemm_bf16_red(
        ctypes.c_void_p(a_ptr), lda, a_mn, ctypes.c_void_p(b_ptr), ldb, b_mn,
        ctypes.c_void_p(out.data_ptr()), out.stride(0), int(out.dtype == torch.float32),
        M, N, K, float(alpha), ctypes.c_void_p(red_buf.data_ptr()),
        ctypes.c_void_p(red_row.data_ptr()), _lib.ptr_array(red_bases), len(red_bases),
        int(red_ld), FUSED_MODES[mode], ctypes.c_void_p(stream.cuda_stream)),
        "ntp_gemm_bf16_red")


def partner_row_map(cols, partner_cols, device):
    """For a shard whose rows are units `cols`, the (buffer, row) of each unit in
    the partner replica's per-rank layout `partner_cols` (list of arrays)."""
    k = int(max(max(c.max() for c in partner_cols if len(c)), np.max(cols))) + 1
    owner = np.full(k, -1, dtype=np.int32)
    pos = np.zeros(k, dtype=np.int32)
    for r, c in enumerate(partner_cols):
        owner[c] = r
        pos[c] = np.arange(len(c), dtype=np.int32)
    cols = np.asarray(cols)
    return (torch.from_numpy(owner[cols]).to(device), torch.from_numpy(pos[cols]).to(device))


_NO_PARTNER: dict = {}


def _no_partner_rows(M: int, device) -> tuple:
    """(red_buf, red_row) row maps with no partner copy (-1), cached per (M, device)."""
    key = (M, str(device))
    if key not in _NO_PARTNER:
        _NO_PARTNER[key] = (torch.full((M,), -1, dtype=torch.int32, device=device),
                            torch.zeros((M,), dtype=torch.int32, device=device))
    return _NO_PARTNER[key]


def _pad8(n: int) -> int:
    return (n + 7) // 8 * 8


class MlpShard:
    """One TP rank's slice of an MLP block: unit-major bf16 weights [n, 2, h]."""

    def __init__(self, A: np.ndarray, B: np.ndarray, cols, device="cuda"):
        cols = np.asarray(cols, dtype=np.int64)
        h = A.shape[0]
        w = np.empty((len(cols), 2, h))
        w[:, 0, :] = A[:, cols].T
        w[:, 1, :] = B[cols, :]
        self.n, self.h = len(cols), h
        self.W = torch.from_numpy(w).to(device=device, dtype=torch.bfloat16)
        self.H = self.Y = None

    def activations(self, X: torch.Tensor) -> None:
        """H = X A_i and Y = GeLU(H) (one GEMM, fused GeLU epilogue) -- what
        backward() needs from the forward pass."""
        T = X.shape[0]
        npad = _pad8(self.n)
        if self.H is None or self.H.shape[0] != T:
            self.H = torch.empty((T, npad), dtype=torch.bfloat16, device=X.device)
            self.Y = torch.empty((T, npad), dtype=torch.bfloat16, device=X.device)
        mm(X, self.W[:, 0, :], self.Y[:, :self.n], epilogue="gelu", aux=self.H[:, :self.n])

    def forward(self, X: torch.Tensor, Z: torch.Tensor, accumulate: bool = False) -> None:
        """H = X A_i, Y = GeLU(H) (fused epilogue), Z (+)= Y B_i (fp32 partial)."""
        T = X.shape[0]
        self.activations(X)
        Y = self.Y[:, :self.n]
        if accumulate and self.h % 32 == 0 and Z.dtype == torch.float32 and Z.is_contiguous():
            # Z += Y B_i inside the GEMM: the epilogue adds each staged box into Z
            # with a TMA bulk reduction (ntp_gemm_bf16_red mode 3, no partner
            # copy: every row's partner index is -1).  Each element gets one
            # add, so the ordered sum is exactly Z + part, as the eager add was.
            rb, rr = _no_partner_rows(T, X.device)
            mm_red(Y, self.W[:, 1, :].T, Z, 1.0, rb, rr, [], self.h, mode="red_tma")
        elif accumulate:
            part = torch.empty((T, self.h), dtype=torch.float32, device=X.device)
            mm(Y, self.W[:, 1, :].T, part)
            Z += part
        else:
            mm(Y, self.W[:, 1, :].T, Z)

    def backward(self, X: torch.Tensor, G: torch.Tensor, grads: torch.Tensor,
                 pdl: str | None = None, alpha: float = 1.0) -> None:
        """Weight gradients written unit-major into grads [n, 2, h] (bf16 or fp32):
        grads[:, 1, :] = alpha * Y^T G, grads[:, 0, :] = alpha * D^T X with
        D = (G B_i^T) * GeLU'(H).  alpha folds a replica's batch weight into the
        wgrad epilogue (aligned regions then sync with a plain SUM, no scale pass).

        pdl: chain the three GEMMs with programmatic dependent launch.  The
        first GEMM takes this mode ("after", or "independent" when the caller
        knows the previous kernel of the stream shares no data with it); dB,
        which does not read D, runs "independent" under its tail; dA waits
        ("after").  D is then a per-shard buffer, never a recycled temporary
        a still-running GEMM could be reading."""
        T = X.shape[0]
        H, Y = self.H[:, :self.n], self.Y[:, :self.n]
        if pdl is None:
            Dfull = torch.empty((T, _pad8(self.n)), dtype=torch.bfloat16, device=X.device)
        else:
            if getattr(self, "_D", None) is None or self._D.shape[0] != T:
                self._D = torch.empty((T, _pad8(self.n)), dtype=torch.bfloat16, device=X.device)
            Dfull = self._D
        D = Dfull[:, :self.n]
        mm(G, self.W[:, 1, :], D, epilogue="dgelu", aux=H, pdl=pdl)
        mm(Y.T, G.T, grads[:, 1, :], alpha=alpha, pdl=None if pdl is None else "independent")
        mm(D.T, X.T, grads[:, 0, :], alpha=alpha, pdl=None if pdl is None else "after")

    def backward_synced(self, X: torch.Tensor, G: torch.Tensor, grads: torch.Tensor, alpha: float,
                        red_buf: torch.Tensor, red_row: torch.Tensor, partner_arenas,
                        stream=None, mode: str = "red") -> None:
        """backward() with the NTP sync fused into the weight-gradient epilogues:
        alpha * dB, alpha * dA^T go into this rank's unit-major arena and into the
        partner replica's arenas -- red.add into zeroed arenas (mode "red"), or
        stores into the partner's staging arenas (mode "push", finished by
        ``finish_push``).  Afterwards both replicas hold w_h*g_h + w_r*g_r."""
        T = X.shape[0]
        H, Y = self.H[:, :self.n], self.Y[:, :self.n]
        Dfull = torch.empty((T, _pad8(self.n)), dtype=torch.bfloat16, device=X.device)
        D = Dfull[:, :self.n]
        mm(G, self.W[:, 1, :], D, epilogue="dgelu", aux=H, stream=stream)
        eb = grads.element_size()
        h = self.h
        bases_b = [int(t.data_ptr()) + h * eb for t in partner_arenas]
        bases_a = [int(t.data_ptr()) for t in partner_arenas]
        mm_red(Y.T, G.T, grads[:, 1, :], alpha, red_buf, red_row, bases_b, 2 * h, stream, mode)
        mm_red(D.T, X.T, grads[:, 0, :], alpha, red_buf, red_row, bases_a, 2 * h, stream, mode)


_FINISH_PLANS: dict = {}


def finish_push(arena: torch.Tensor, staging: torch.Tensor, stream=None) -> None:
    """arena += staging (fp32 accumulation, arena operand first on both replicas'
    sides so the two copies add the same two terms) -- the local tail of the
    "push" fused sync, after the partners' done signal."""
    from .plans import OPS, Plan, dtype_code
    n, dt, dev = arena.numel(), arena.dtype, arena.device.index
    key = (n, dt, dev)
    plan = _FINISH_PLANS.get(key)
    if plan is None:
        plan = Plan(dtype_code(dt)).add_units(n, [0], [0], [1], [0]).finalize().upload(dev)
        _FINISH_PLANS[key] = plan
    plan.grad_sync_into([arena.data_ptr(), staging.data_ptr()], OPS["sum"], 1.0, 1.0, 1, stream)


def mlp_forward_tp(X: torch.Tensor, shards) -> torch.Tensor:
    """Z = sum_i GeLU(X A_i) B_i in ascending rank order (tpnumerics.py:177-185);
    on one GPU the TP all-reduce is this ordered sum."""
    Z = torch.zeros((X.shape[0], shards[0].h), dtype=torch.float32, device=X.device)
    for i, sh in enumerate(shards):
        sh.forward(X, Z, accumulate=i > 0)
    return Z


def mlp_backward_tp(X: torch.Tensor, shards, G: torch.Tensor, replica) -> None:
    """Parameter gradients of every rank straight into ``replica.grads`` (the
    unit-major arenas of a tpnumerics.MlpReplica built on the same columns)."""
    for sh, g in zip(shards, replica.grads):
        if tuple(g.shape) != (sh.n, 2, sh.h):
            raise ValueError("replica layout does not match the shards")
        sh.backward(X, G, g)
    replica._has_grads = True
