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
    """One MLP block, A [hidden x ffn], B [ffn x hidden] (tpnumerics.py:40-67)."""

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
    (``set_grads`` or ``mlp_backward_tp``), as in the reference.  The default
    gradient dtype is float64, the reference's (its inputs are cast up,
    tpnumerics.py:47-48), so the reference's own call sites keep their 1e-12
    tolerances; bf16 / fp32 replicas are the training-time layouts.
    """

    def __init__(self, layer: MlpLayer, assignment, *, dtype: torch.dtype = torch.float64,
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
    def a_frags(self) -> list[np.ndarray]:
        """Per-rank weight fragments A[:, cols_r] [hidden, n_r] (tpnumerics.py:141)."""
        return [self.layer.A[:, c] for c in self.cols]

    @property
    def b_frags(self) -> list[np.ndarray]:
        """Per-rank weight fragments B[cols_r, :] [n_r, hidden] (tpnumerics.py:142)."""
        return [self.layer.B[c, :] for c in self.cols]

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
# dense / TP forward and backward (tpnumerics.py:25-36, 168-252), on the device.
# Inputs may be numpy arrays (the reference's callers) or tensors; numpy in,
# numpy out.  float64 work runs as fp64 device math (bit-for-bit the same
# formulas, BLAS-order differences only, <= 1e-12 like the reference's own
# tolerances); bf16 replicas run the tcgen05 GEMMs of linear.py.


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_06095_b200 computes on a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _dev64(x, device=None) -> torch.Tensor:
    dev = _device() if device is None else device
    if torch.is_tensor(x):
        return x.to(device=dev, dtype=torch.float64)
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=dev)


def _out(t: torch.Tensor, like):
    return t if torch.is_tensor(like) else t.cpu().numpy()


def _gelu_t(x):
    # GELU_C read at call time: a caller that patches the module constant (the
    # reference's drift test, test_tpnumerics.py / cli verify --suite golden)
    # sees the change, as with the reference's gelu
    return 0.5 * x * (1.0 + torch.tanh(SQRT_2_OVER_PI * (x + GELU_C * x**3)))


def _gelu_grad_t(x):
    u = SQRT_2_OVER_PI * (x + GELU_C * x**3)
    t = torch.tanh(u)
    du = SQRT_2_OVER_PI * (1.0 + 3.0 * GELU_C * x**2)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t**2) * du


def gelu(x):
    """tanh-approximation GeLU (tpnumerics.py:25-28), float64."""
    return _out(_gelu_t(_dev64(x)), x)


def gelu_grad(x):
    """d GeLU / dx (tpnumerics.py:31-36), float64."""
    return _out(_gelu_grad_t(_dev64(x)), x)


def _check_features(X, hidden: int) -> None:
    if X.shape[1] != hidden:
        raise ValueError(f"X has {X.shape[1]} features, layer expects {hidden}")


def mlp_forward_dense(X, layer: MlpLayer):
    """Z = GeLU(X A) B (tpnumerics.py:170-174)."""
    Xd = _dev64(X)
    _check_features(Xd, layer.hidden)
    return _out(_gelu_t(Xd @ _dev64(layer.A)) @ _dev64(layer.B), X)


def _shards(replica: MlpReplica):
    """tcgen05 weight shards (unit-major bf16) of a replica, built once."""
    from .linear import MlpShard
    sh = getattr(replica, "_shards", None)
    if sh is None:
        sh = [MlpShard(replica.layer.A, replica.layer.B, c, device=replica.device)
              for c in replica.cols]
        replica._shards = sh
    return sh


def mlp_forward_tp(X, replica: MlpReplica):
    """Sum of the per-rank partial outputs GeLU(X A_r) B_r in ascending rank
    order (tpnumerics.py:177-185).  bf16 replicas: the tcgen05 column- then
    row-parallel GEMMs (bf16 operands, fp32 partial sums; linear.py);
    otherwise float64."""
    Xd = _dev64(X, replica.device)
    _check_features(Xd, replica.hidden)
    if replica.dtype == torch.bfloat16:
        from .linear import mlp_forward_tp as fwd
        return _out(fwd(Xd.to(torch.bfloat16), _shards(replica)).double(), X)
    A, B = _dev64(replica.layer.A, replica.device), _dev64(replica.layer.B, replica.device)
    Z = torch.zeros((Xd.shape[0], replica.hidden), dtype=torch.float64, device=replica.device)
    for cols in replica.cols:
        idx = torch.as_tensor(cols, device=replica.device)
        Z += _gelu_t(Xd @ A[:, idx]) @ B[idx, :]
    return _out(Z, X)


def mlp_backward(X, layer: MlpLayer, upstream_grad):
    """Dense parameter gradients (dA [h, ffn], dB [ffn, h]) of Z = GeLU(X A) B
    (tpnumerics.py:220-235): dB = GeLU(XA)^T G, dA = X^T((G B^T) * GeLU'(XA))."""
    Xd, G = _dev64(X), _dev64(upstream_grad)
    if tuple(G.shape) != (Xd.shape[0], layer.hidden):
        raise ValueError(f"upstream grad shape {tuple(G.shape)} != {(Xd.shape[0], layer.hidden)}")
    A, B = _dev64(layer.A), _dev64(layer.B)
    H = Xd @ A
    dB = _gelu_t(H).T @ G
    dA = Xd.T @ ((G @ B.T) * _gelu_grad_t(H))
    return _out(dA, X), _out(dB, X)


def mlp_backward_tp(X, replica: MlpReplica, upstream_grad) -> None:
    """Per-rank dB_r = GeLU(X A_r)^T G, dA_r = X^T((G B_r^T) * GeLU'(X A_r))
    (tpnumerics.py:238-252), stored unit-major in the replica's arenas.

    bf16 replicas run the tcgen05 GEMMs (linear.MlpShard: forward for H/Y, then
    the dGeLU and the two weight-gradient GEMMs writing the arena in place);
    fp32 / fp64 replicas are computed in float64 and stored in their dtype."""
    dev = replica.device
    if replica.dtype == torch.bfloat16:
        Xb = _dev64(X, dev).to(torch.bfloat16)
        Gb = _dev64(upstream_grad, dev).to(torch.bfloat16)
        for sh, g in zip(_shards(replica), replica.grads):
            sh.activations(Xb)
            sh.backward(Xb, Gb, g)
        replica._has_grads = True
        return
    Xd, G = _dev64(X, dev), _dev64(upstream_grad, dev)
    A, B = _dev64(replica.layer.A, dev), _dev64(replica.layer.B, dev)
    for g, cols in zip(replica.grads, replica.cols):
        idx = torch.as_tensor(cols, device=dev)
        A_i, B_i = A[:, idx], B[idx, :]
        H_i = Xd @ A_i
        g[:, 1, :].copy_((_gelu_t(H_i).T @ G).to(replica.dtype))
        g[:, 0, :].copy_((Xd.T @ ((G @ B_i.T) * _gelu_grad_t(H_i))).T.to(replica.dtype))
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


class _HostPath:
    """Device resources of the reference-object path for one (layout, hidden):
    the fp64 plan (built and uploaded once), the unit-major device arenas and
    per-fragment device staging, all reused call after call.  The reference's
    fragments are copied to and from the device as they lie (grad_a [h, n_r]
    and grad_b [n_r, h], C-contiguous): the A-half transposes run on the device
    and the results land straight in the caller's arrays -- no host-side
    restaging."""

    def __init__(self, healthy, reduced, k: int, device: torch.device):
        h = healthy.layer.hidden
        self.h = h
        self.device = device
        plan = build_pair_plan(healthy.cols, reduced.cols, k, 2 * h, _lib.NTP_F64)
        self.plan = plan.finalize().upload(device.index)
        sizes = [len(c) for c in list(healthy.cols) + list(reduced.cols)]
        self.dev = [torch.empty((n, 2 * h), dtype=torch.float64, device=device) for n in sizes]
        self.ga = [torch.empty((h, n), dtype=torch.float64, device=device) for n in sizes]
        self.ptrs = tensor_ptrs(self.dev)
        self.stream = torch.cuda.Stream(device)
        self.bytes = sum(n * 2 * h * 8 for n in sizes)

    def run(self, healthy, reduced, code, w_h, w_r) -> None:
        h = self.h
        frags = [(ga, gb) for rep in (healthy, reduced) for ga, gb in zip(rep.grad_a, rep.grad_b)]
        host = [(torch.from_numpy(np.ascontiguousarray(ga, dtype=np.float64)),
                 torch.from_numpy(np.ascontiguousarray(gb, dtype=np.float64))) for ga, gb in frags]
        s = self.stream
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for d, ga_d, (ga, gb) in zip(self.dev, self.ga, host):
                ga_d.copy_(ga)                    # [h, n_r] as the caller holds it
                d[:, h:].copy_(gb)                # B rows: already unit-major
                d[:, :h].copy_(ga_d.T)            # A columns -> unit-major, on the device
            self.plan.grad_sync(self.ptrs, code, w_h, w_r, s)
            for d, ga_d in zip(self.dev, self.ga):
                ga_d.copy_(d[:, :h].T)
        for (ga, gb), (ga_t, gb_t), d, ga_d in zip(frags, host, self.dev, self.ga):
            with torch.cuda.stream(s):
                ga_t.copy_(ga_d)                  # device -> the caller's memory
                gb_t.copy_(d[:, h:])
            s.synchronize()
            if ga_t.data_ptr() != np.asarray(ga).__array_interface__["data"][0]:
                ga[...] = ga_t.numpy()            # the caller's array was not contiguous fp64
            if gb_t.data_ptr() != np.asarray(gb).__array_interface__["data"][0]:
                gb[...] = gb_t.numpy()


_HOST_PATHS: dict = {}


def _nonuniform_host(healthy, reduced, smap, code, w_h, w_r) -> None:
    """Reference-object path (numpy fp64 fragments in the reference's shapes,
    mutated in place like tpnumerics.py:346-356): pinned staging -> one H2D per
    rank -> the fp64 sync kernel -> D2H -> the caller's arrays.  The plan, the
    pinned staging and the device arenas are cached per layout, so repeated
    calls (a training loop) allocate nothing.  fp64 keeps the result bit-exact
    with the reference for op sum/mean."""
    dev = torch.device("cuda", torch.cuda.current_device())
    key = (tuple(c.tobytes() for c in healthy.cols), tuple(c.tobytes() for c in reduced.cols),
           healthy.layer.hidden, smap.k, dev.index)
    path = _HOST_PATHS.get(key)
    if path is None:
        if len(_HOST_PATHS) > 16:
            _HOST_PATHS.clear()
        path = _HOST_PATHS[key] = _HostPath(healthy, reduced, smap.k, dev)
    path.run(healthy, reduced, code, w_h, w_r)


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


@dataclass(frozen=True)
class AttentionLayer:
    """Multi-head attention weights (tpnumerics.py:70-112): wq/wk/wv
    [H, hidden, head_dim], wo [H, head_dim, hidden], float64."""

    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray

    def __post_init__(self):
        for name in ("wq", "wk", "wv", "wo"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        if not (self.wq.shape == self.wk.shape == self.wv.shape):
            raise ValueError("wq/wk/wv shapes differ")
        H, hidden, head_dim = self.wq.shape
        if self.wo.shape != (H, head_dim, hidden):
            raise ValueError(f"wo shape {self.wo.shape} != {(H, head_dim, hidden)}")

    @property
    def heads(self) -> int:
        return self.wq.shape[0]

    @property
    def hidden(self) -> int:
        return self.wq.shape[1]

    @property
    def head_dim(self) -> int:
        return self.wq.shape[2]

    @classmethod
    def random(cls, heads: int, hidden: int, head_dim: int, seed: int = 0) -> "AttentionLayer":
        """Seeded N(0,1) draws in the reference's order: wq, wk, wv, wo."""
        rng = np.random.default_rng(seed)
        shapes = [(heads, hidden, head_dim)] * 3 + [(heads, head_dim, hidden)]
        return cls(*(rng.standard_normal(s) for s in shapes))


def _heads_output(X: torch.Tensor, layer: AttentionLayer, heads) -> torch.Tensor:
    """sum over `heads` of softmax(Q K^T / sqrt(d)) V W_o (tpnumerics.py:188-199),
    all heads of the set batched, float64."""
    idx = torch.as_tensor(np.asarray(heads, dtype=np.int64), device=X.device)
    wq, wk, wv, wo = (_dev64(w, X.device)[idx] for w in (layer.wq, layer.wk, layer.wv, layer.wo))
    Q, K, V = (torch.einsum("th,nhd->ntd", X, w) for w in (wq, wk, wv))
    P = torch.softmax(Q @ K.transpose(1, 2) / np.sqrt(layer.head_dim), dim=-1)
    out = torch.zeros((X.shape[0], layer.hidden), dtype=torch.float64, device=X.device)
    for o in torch.bmm(P @ V, wo):  # ascending head order, as the reference
        out += o
    return out


def attention_forward_dense(X, layer: AttentionLayer):
    """Sum of every head's output (tpnumerics.py:202-207), float64."""
    return _out(_heads_output(_dev64(X), layer, np.arange(layer.heads)), X)


def attention_forward_tp(X, replica):
    """Per-rank partial sums over owned heads, ranks in ascending order
    (tpnumerics.py:210-217), float64."""
    Xd = _dev64(X)
    Z = torch.zeros((Xd.shape[0], replica.layer.hidden), dtype=torch.float64, device=Xd.device)
    for owned in replica.heads:
        if len(owned):
            Z += _heads_output(Xd, replica.layer, owned)
    return _out(Z, X)


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
