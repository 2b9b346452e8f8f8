"""Tensor-parallel gradient sync with the reference's API, executed on B200.

Drop-in for the sync half of ``ntpsim.tpnumerics`` (pkg/src/ntpsim/
tpnumerics.py): ``MlpLayer``, ``MlpReplica``, the assignment helpers,
``uniform_grad_sync`` and ``nonuniform_grad_sync`` keep their names, argument
meaning, in-place semantics and ValueError texts.  What changes is where the
gradients live: an ``MlpReplica`` here stores each rank's gradient fragment in
device memory, unit-major ([n_r, 2, hidden]: unit p = A column p ; B row p),
and exposes the reference's shapes as views: ``grad_a[r]`` is [hidden, n_r]
and ``grad_b[r]`` is [n_r, hidden].

``nonuniform_grad_sync`` additionally accepts the reference's own numpy-backed
``MlpReplica`` objects: the gradients then travel host -> device -> host
around the same kernel (the end-to-end path bench.py times as ``e2e``).

Extension beyond the reference: ``weights=(w_h, w_r)`` applies per-replica
batch weighting, ``w_h*g_h + w_r*g_r``; (1, 1) equals op "sum" and
(1/2, 1/2) equals op "mean".
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .plans import OPS, Plan, dtype_code, layout_offsets, tensor_ptrs
from .shardmap import ShardMap

GELU_C = 0.044715                              # tpnumerics.py:21
SQRT_2_OVER_PI = float(np.sqrt(2.0 / np.pi))   # tpnumerics.py:22


@dataclass(frozen=True)
class MlpLayer:
    """One MLP block, A [hidden x ffn], B [ffn x hidden] (tpnumerics.py:39-67)."""

    A: np.ndarray
    B: np.ndarray

    def __post_init__(self):
        A = np.asarray(self.A, dtype=np.float64)
        B = np.asarray(self.B, dtype=np.float64)
        if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0] or A.shape[0] != B.shape[1]:
            raise ValueError(f"inconsistent MLP shapes {A.shape} / {B.shape}")
        object.__setattr__(self, "A", A)
        object.__setattr__(self, "B", B)

    @property
    def hidden(self) -> int:
        return self.A.shape[0]

    @property
    def ffn(self) -> int:
        return self.A.shape[1]

    @classmethod
    def random(cls, hidden: int, ffn: int | None = None, seed: int = 0) -> "MlpLayer":
        ffn = 4 * hidden if ffn is None else ffn
        rng = np.random.default_rng(seed)
        A = rng.standard_normal((hidden, ffn))
        return cls(A=A, B=rng.standard_normal((ffn, hidden)))


def contiguous_assignment(k: int, n: int) -> list[np.ndarray]:
    """Balanced contiguous split, remainder first (tpnumerics.py:115-120)."""
    sizes = k // n + (np.arange(n) < k % n)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    return [np.arange(bounds[i], bounds[i + 1], dtype=np.int64) for i in range(n)]


def assignment_from_comp(smap: ShardMap) -> list[np.ndarray]:
    return [smap.comp_columns(r) for r in range(smap.n1)]


def assignment_from_sync(smap: ShardMap) -> list[np.ndarray]:
    return [smap.sync_columns(r) for r in range(smap.n2)]


class MlpReplica:
    """One TP replica: per-rank columns and device-resident unit-major gradients.

    Mirrors tpnumerics.py:131-155.  ``grads[r]`` is the [n_r, 2, hidden]
    device tensor; ``grad_a``/``grad_b`` are None until gradients are set
    (``set_grads`` or ``mlp_backward_tp``), as in the reference.
    """

    def __init__(self, layer: MlpLayer, assignment, *, dtype: torch.dtype = torch.float32,
                 device: int | str | torch.device | None = None):
        cols = np.concatenate([np.asarray(a, dtype=np.int64) for a in assignment])
        if len(cols) != layer.ffn or len(np.unique(cols)) != layer.ffn:
            raise ValueError("assignment does not partition the ffn columns exactly once")
        self.layer = layer
        self.n = len(assignment)
        self.cols = [np.asarray(a, dtype=np.int64) for a in assignment]
        self.dtype = dtype
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("MlpReplica gradients live on a CUDA device")
        h = layer.hidden
        self.grads = [torch.zeros((len(c), 2, h), dtype=dtype, device=self.device)
                      for c in self.cols]
        self._has_grads = False

    @property
    def hidden(self) -> int:
        return self.layer.hidden

    @property
    def grad_a(self):
        if not self._has_grads:
            return None
        return [g[:, 0, :].T for g in self.grads]   # [hidden, n_r] views

    @property
    def grad_b(self):
        if not self._has_grads:
            return None
        return [g[:, 1, :] for g in self.grads]     # [n_r, hidden] views

    def set_grads(self, grad_a, grad_b) -> "MlpReplica":
        """Load per-rank fragments in the reference's shapes ([h, n_r], [n_r, h])."""
        if len(grad_a) != self.n or len(grad_b) != self.n:
            raise ValueError("one gradient fragment per rank is required")
        for g, ga, gb in zip(self.grads, grad_a, grad_b):
            ga = torch.as_tensor(np.asarray(ga) if not torch.is_tensor(ga) else ga)
            gb = torch.as_tensor(np.asarray(gb) if not torch.is_tensor(gb) else gb)
            g[:, 0, :].copy_(ga.T.to(self.device, self.dtype))
            g[:, 1, :].copy_(gb.to(self.device, self.dtype))
        self._has_grads = True
        return self

    def set_units(self, units) -> "MlpReplica":
        """Load per-rank unit-major arrays ([n_r, 2h] or flat)."""
        for g, u in zip(self.grads, units):
            t = u if torch.is_tensor(u) else torch.from_numpy(np.ascontiguousarray(u))
            g.view(-1).copy_(t.reshape(-1).to(self.device, self.dtype))
        self._has_grads = True
        return self

    def units(self) -> list[np.ndarray]:
        """Per-rank unit-major fragments as float64 numpy [n_r, 2h]."""
        return [g.reshape(g.shape[0], -1).to(torch.float64).cpu().numpy() for g in self.grads]

    def dense_grads(self) -> tuple[np.ndarray, np.ndarray]:
        """Reassemble dense dA [h, ffn], dB [ffn, h] as float64 (tpnumerics.py:146-155)."""
        if not self._has_grads:
            raise ValueError("replica holds no gradients")
        h = self.hidden
        dA = np.zeros((h, self.layer.ffn))
        dB = np.zeros((self.layer.ffn, h))
        for cols, u in zip(self.cols, self.units()):
            dA[:, cols] = u[:, :h].T
            dB[cols, :] = u[:, h:]
        return dA, dB


# ---------------------------------------------------------------------------
# gradient producer (device).  The weight-gradient GEMMs of tpnumerics.py:238-252
# written straight into the unit-major layout the sync consumes.


def _gelu_t(x):
    return 0.5 * x * (1.0 + torch.tanh(SQRT_2_OVER_PI * (x + GELU_C * x**3)))


def _gelu_grad_t(x):
    u = SQRT_2_OVER_PI * (x + GELU_C * x**3)
    t = torch.tanh(u)
    du = SQRT_2_OVER_PI * (1.0 + 3.0 * GELU_C * x**2)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t**2) * du


def mlp_backward_tp(X, replica: MlpReplica, upstream_grad) -> None:
    """Per-rank dB_r = GeLU(X A_r)^T G, dA_r = X^T((G B_r^T) * GeLU'(X A_r))
    (tpnumerics.py:238-252), computed on the replica's device in fp64 and
    stored unit-major in the replica's gradient dtype."""
    dev = replica.device
    X = torch.as_tensor(np.asarray(X, dtype=np.float64), device=dev)
    G = torch.as_tensor(np.asarray(upstream_grad, dtype=np.float64), device=dev)
    A = torch.as_tensor(replica.layer.A, device=dev)
    B = torch.as_tensor(replica.layer.B, device=dev)
    for g, cols in zip(replica.grads, replica.cols):
        idx = torch.as_tensor(cols, device=dev)
        A_i, B_i = A[:, idx], B[idx, :]
        H_i = X @ A_i
        g[:, 1, :].copy_((_gelu_t(H_i).T @ G).to(replica.dtype))
        g[:, 0, :].copy_((X.T @ ((G @ B_i.T) * _gelu_grad_t(H_i))).T.to(replica.dtype))
    replica._has_grads = True


# ---------------------------------------------------------------------------
# syncs


def _op_and_weights(op: str, weights):
    if op not in ("sum", "mean"):
        raise ValueError(f"unknown reduction op {op!r}")
    if weights is None:
        return OPS[op], 1.0, 1.0
    if op != "sum":
        raise ValueError("weights= replaces op; pass op='sum' with explicit weights")
    w_h, w_r = (float(w) for w in weights)
    return OPS["weighted"], w_h, w_r


def _validate_nonuniform(healthy, reduced, smap: ShardMap) -> None:
    """The reference's checks and messages, tpnumerics.py:299-312."""
    if healthy.n != smap.n1 or reduced.n != smap.n2:
        raise ValueError(
            f"replica degrees ({healthy.n}, {reduced.n}) do not match map ({smap.n1}, {smap.n2})"
        )
    if healthy.layer.ffn != smap.k:
        raise ValueError(f"map is over k={smap.k} columns, layer has ffn={healthy.layer.ffn}")
    for r in range(smap.n1):
        if not np.array_equal(np.sort(healthy.cols[r]), smap.comp_columns(r)):
            raise ValueError("healthy replica is not sharded by the map's comp layout")
    for r in range(smap.n2):
        if not np.array_equal(np.sort(reduced.cols[r]), smap.sync_columns(r)):
            raise ValueError("reduced replica is not sharded by the map's sync layout")
    if healthy.grad_a is None or reduced.grad_a is None:
        raise ValueError("both replicas must hold gradients")


def build_pair_plan(h_cols, r_cols, k: int, unit: int, dtype: int, *, h_base=None, r_base=None,
                    h_bufs=None, r_bufs=None, plan: Plan | None = None) -> Plan:
    """Append one segment (k units of `unit` elements) pairing the healthy
    layout h_cols with the reduced layout r_cols.  Buffer indices default to
    healthy ranks 0..n1-1 and reduced ranks n1..n1+n2-1 (1-GPU emulation)."""
    h_owner, h_off = layout_offsets(h_cols, k, unit, h_base)
    r_owner, r_off = layout_offsets(r_cols, k, unit, r_base)
    h_map = np.arange(len(h_cols)) if h_bufs is None else np.asarray(h_bufs)
    r_map = len(h_cols) + np.arange(len(r_cols)) if r_bufs is None else np.asarray(r_bufs)
    plan = Plan(dtype) if plan is None else plan
    plan.add_units(unit, h_map[h_owner], h_off, r_map[r_owner], r_off)
    return plan


_PLAN_CACHE: dict = {}


def _cached_pair_plan(healthy: MlpReplica, reduced: MlpReplica) -> Plan:
    dev = healthy.device.index if healthy.device.index is not None else torch.cuda.current_device()
    key = (tuple(c.tobytes() for c in healthy.cols), tuple(c.tobytes() for c in reduced.cols),
           healthy.hidden, healthy.dtype, dev)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = build_pair_plan(healthy.cols, reduced.cols, healthy.layer.ffn, 2 * healthy.hidden,
                               dtype_code(healthy.dtype)).finalize().upload(dev)
        if len(_PLAN_CACHE) > 64:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = plan
    return plan


def nonuniform_grad_sync(healthy, reduced, smap: ShardMap, op: str = "sum",
                         weights=None) -> None:
    """Gradient sync between an n1-way and an n2-way replica, in place
    (tpnumerics.py:289-356), as ONE device kernel: each unit is read from its
    healthy owner and its reduced owner, reduced (healthy operand first, fp32
    accumulation), and written back to both owners."""
    _validate_nonuniform(healthy, reduced, smap)
    code, w_h, w_r = _op_and_weights(op, weights)
    if not isinstance(healthy, MlpReplica) or not isinstance(reduced, MlpReplica):
        return _nonuniform_host(healthy, reduced, smap, code, w_h, w_r)
    if healthy.dtype != reduced.dtype or healthy.device != reduced.device:
        raise ValueError("replicas must share gradient dtype and device")
    plan = _cached_pair_plan(healthy, reduced)
    plan.grad_sync(tensor_ptrs(healthy.grads + reduced.grads), code, w_h, w_r)


def _nonuniform_host(healthy, reduced, smap, code, w_h, w_r) -> None:
    """Reference-object path: numpy fp64 fragments in, numpy fragments out (in
    place), H2D + kernel + D2H.  fp64 keeps parity with the reference bit-exact
    for op sum/mean."""
    h = healthy.layer.hidden
    dev = torch.device("cuda", torch.cuda.current_device())
    bufs = []
    for rep in (healthy, reduced):
        for ga, gb in zip(rep.grad_a, rep.grad_b):
            u = np.concatenate([np.asarray(ga).T, np.asarray(gb)], axis=1)
            bufs.append(torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64))
                        .pin_memory().to(dev, non_blocking=True))
    plan = build_pair_plan(healthy.cols, reduced.cols, smap.k, 2 * h, _lib.NTP_F64)
    plan.finalize().upload(dev.index)
    plan.grad_sync(tensor_ptrs(bufs), code, w_h, w_r)
    outs = [b.cpu().numpy() for b in bufs]
    i = 0
    for rep in (healthy, reduced):
        for ga, gb in zip(rep.grad_a, rep.grad_b):
            ga[...] = outs[i][:, :h].T
            gb[...] = outs[i][:, h:]
            i += 1


def uniform_grad_sync(replicas, op: str = "sum", weights=None) -> None:
    """Shard-by-shard reduction across identically sharded replicas, in place
    (tpnumerics.py:263-286): "sum" in replica order, "mean" a true mean over
    all replicas; ``weights`` (one per replica) is the weighted extension."""
    first = replicas[0]
    for r in replicas[1:]:
        if r.n != first.n or any(not np.array_equal(a, b) for a, b in zip(r.cols, first.cols)):
            raise ValueError("replicas are not identically sharded")
    for rep in replicas:
        if rep.grad_a is None:
            raise ValueError("replica holds no gradients")
    if op not in ("sum", "mean"):
        raise ValueError(f"unknown reduction op {op!r}")
    code = OPS[op]
    w = None
    if weights is not None:
        if op != "sum" or len(weights) != len(replicas):
            raise ValueError("weights= needs op='sum' and one weight per replica")
        code, w = OPS["weighted"], (np.ascontiguousarray(weights, dtype=np.float64))
    L = _lib.load()
    for rank in range(first.n):
        ts = [rep.grads[rank] for rep in replicas]
        stream = torch.cuda.current_stream(ts[0].device)
        wp = None if w is None else w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        _lib.check(L.ntp_uniform_sync(_lib.ptr_array(tensor_ptrs(ts)), len(ts), ts[0].numel(),
                                      dtype_code(first.dtype), code, wp,
                                      ctypes.c_void_p(stream.cuda_stream)),
                   "ntp_uniform_sync")


def multi_grad_sync(replicas, op: str = "sum", weights=None) -> None:
    """DP > 2 sync across replicas of ANY layouts (healthy TP-n and degraded
    TP-m mixed), in place: every unit ends as the reduction of its R copies in
    replica order -- uniform_grad_sync's "sum"/"mean" semantics
    (tpnumerics.py:263-286) over nonuniform_grad_sync's layouts (289-356), or
    the batch-weighted sum with ``weights`` (one per replica).  One kernel reads
    each copy once and writes the result into every owner."""
    from .plans import MultiPlan
    first = replicas[0]
    if len(replicas) < 2:
        raise ValueError("need at least two replicas")
    for rep in replicas:
        if rep.grad_a is None:
            raise ValueError("replica holds no gradients")
        if rep.layer.ffn != first.layer.ffn or rep.hidden != first.hidden:
            raise ValueError("replicas hold different layers")
        if not isinstance(rep, MlpReplica) or rep.dtype != first.dtype or rep.device != first.device:
            raise ValueError("replicas must be device MlpReplicas of one dtype and device")
    if op not in ("sum", "mean"):
        raise ValueError(f"unknown reduction op {op!r}")
    code = OPS[op]
    if weights is not None:
        if op != "sum" or len(weights) != len(replicas):
            raise ValueError("weights= needs op='sum' and one weight per replica")
        code = OPS["weighted"]
    k, unit = first.layer.ffn, 2 * first.hidden
    bufs, offs, base = [], [], 0
    for rep in replicas:
        owner, off = layout_offsets(rep.cols, k, unit)
        bufs.append(owner + base)
        offs.append(off)
        base += rep.n
    dev = first.device.index if first.device.index is not None else torch.cuda.current_device()
    plan = MultiPlan(dtype_code(first.dtype), len(replicas)).add_units(unit, bufs, offs)
    plan.finalize().upload(dev)
    plan.sync(tensor_ptrs([g for rep in replicas for g in rep.grads]), code, weights)


# ---------------------------------------------------------------------------
# attention heads as sync units.  The reference shards
# attention by whole heads (AttentionReplica, tpnumerics.py:158-167) but has no
# attention gradients; here a head's four blocks (wq, wk, wv: [hidden x hd],
# wo: [hd x hidden]) form one contiguous unit of 4*hidden*hd elements
# (perfmodel.py:270-272) and heads sync exactly like MLP columns.


class AttentionReplica:
    """Per-rank head ownership (tpnumerics.py:158-167) plus device-resident
    head-unit gradients ``grads[r]`` = [n_heads_r, 4, hidden, head_dim] (wo's
    block stored transposed so every head is one contiguous unit)."""

    def __init__(self, layer, head_assignment, *, dtype: torch.dtype = torch.bfloat16,
                 device=None):
        heads = np.concatenate([np.asarray(a, dtype=np.int64) for a in head_assignment])
        if len(heads) != layer.heads or len(np.unique(heads)) != layer.heads:
            raise ValueError("assignment does not partition the heads exactly once")
        self.layer = layer
        self.n = len(head_assignment)
        self.heads = [np.asarray(a, dtype=np.int64) for a in head_assignment]
        self.dtype = dtype
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.unit = 4 * layer.hidden * layer.head_dim
        self.grads = [torch.zeros((len(h), 4, layer.hidden, layer.head_dim), dtype=dtype,
                                  device=self.device) for h in self.heads]
        self._has_grads = False

    def set_units(self, units) -> "AttentionReplica":
        for g, u in zip(self.grads, units):
            t = u if torch.is_tensor(u) else torch.from_numpy(np.ascontiguousarray(u))
            g.view(-1).copy_(t.reshape(-1).to(self.device, self.dtype))
        self._has_grads = True
        return self

    def units(self) -> list[np.ndarray]:
        return [g.reshape(g.shape[0], -1).to(torch.float64).cpu().numpy() for g in self.grads]


def nonuniform_head_sync(healthy: AttentionReplica, reduced: AttentionReplica, smap: ShardMap,
                         op: str = "sum", weights=None) -> None:
    """nonuniform_grad_sync (tpnumerics.py:289-356) over attention heads: the
    shard map is built over k = heads (shardmap.py:141-182, attention_head_partition
    gives the same balanced counts) and every head is one unit."""
    if healthy.n != smap.n1 or reduced.n != smap.n2:
        raise ValueError(
            f"replica degrees ({healthy.n}, {reduced.n}) do not match map ({smap.n1}, {smap.n2})")
    if healthy.layer.heads != smap.k:
        raise ValueError(f"map is over k={smap.k} heads, layer has {healthy.layer.heads}")
    for r in range(smap.n1):
        if not np.array_equal(np.sort(healthy.heads[r]), smap.comp_columns(r)):
            raise ValueError("healthy replica is not sharded by the map's comp layout")
    for r in range(smap.n2):
        if not np.array_equal(np.sort(reduced.heads[r]), smap.sync_columns(r)):
            raise ValueError("reduced replica is not sharded by the map's sync layout")
    if not (healthy._has_grads and reduced._has_grads):
        raise ValueError("both replicas must hold gradients")
    code, w_h, w_r = _op_and_weights(op, weights)
    dev = healthy.device.index if healthy.device.index is not None else torch.cuda.current_device()
    plan = build_pair_plan(healthy.heads, reduced.heads, smap.k, healthy.unit,
                           dtype_code(healthy.dtype)).finalize().upload(dev)
    plan.grad_sync(tensor_ptrs(healthy.grads + reduced.grads), code, w_h, w_r)
