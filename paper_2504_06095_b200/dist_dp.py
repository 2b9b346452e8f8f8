"""DP > 2 with one degraded replica across processes (BASELINE configs[2]:
DP=4 x TP2 with one replica degraded to TP1, batch-proportional weights).

Replicas: m healthy TP-n1 replicas H_0..H_{m-1}, identically laid out (the NTP
comp layout of (k, n1, n2), shardmap.py:141-182), and one degraded TP-n2
replica D (the sync layout).  Every unit must end as

    v = sum_r w_r * g_r        (H replicas and D, replica order H_0.., D)

in all m+1 owners.  The healthy replicas are aligned with each other, so
their part is an NCCL all-reduce; only the D <-> H_0 exchange is nonuniform.
Per step:

  A  H_0's GPUs read D's copy of their units over NVLink and fold it in:
     g_H0 <- w_H0 * g_H0 + w_D * g_D          (ntp_grad_sync_ex, write A only)
  B  NCCL all-reduce of each healthy logical rank across H_0..H_{m-1} with
     per-rank pre-multiplied sums (H_0: 1, H_r: w_Hr) -- no scale kernel
  C  H_0's GPUs push the result into D's arena (ntp_reshard over peer memory)
     and post "done"; D's stream waits for it.

D's link carries S_D*b out (phase A) and S_D*b in (phase C): the one-direction
lower bound for a GPU that must contribute and receive its whole shard.
The oracle for this composition is the reference's uniform_grad_sync
arithmetic on dense layouts (oracle.uniform_sync), as in tests/test_multi.py.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dist import READY, DONE, SIG_BYTES, SIG_WORDS, DeviceOps, _wrap
from .plans import OPS, Plan, dtype_code
from .shardmap import build_shard_map


@dataclass(frozen=True)
class DpPlacement:
    """hp[r][i]: world rank hosting healthy replica r's logical rank i;
    dp[j]: world rank hosting degraded logical rank j."""

    n1: int
    n2: int
    hp: tuple
    dp: tuple

    @classmethod
    def default(cls, world: int, m: int, n1: int, n2: int) -> "DpPlacement":
        need = m * n1 + n2
        if world >= need:  # one logical rank per GPU, spares idle
            hp = tuple(tuple(r * n1 + i for i in range(n1)) for r in range(m))
            return cls(n1, n2, hp, tuple(m * n1 + j for j in range(n2)))
        if world >= m + 1:  # one GPU per healthy replica, the rest for D
            hp = tuple(tuple(r for _ in range(n1)) for r in range(m))
            rest = world - m
            return cls(n1, n2, hp, tuple(m + j * rest // n2 for j in range(n2)))
        raise ValueError(f"DP={m + 1} with one degraded replica needs >= {m + 1} GPUs")


class NtpDpGroup:
    """One process's share of a DP>2 sync: healthy replicas + one degraded."""

    def __init__(self, k: int, unit: int, m: int, plc: DpPlacement, dtype: torch.dtype,
                 device: int, weights, ops: DeviceOps | None = None):
        self.k, self.unit, self.m, self.plc, self.dtype = k, unit, m, plc, dtype
        self.device = device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.ops = ops if ops is not None else DeviceOps(device)
        self.eb = torch.empty(0, dtype=dtype).element_size()
        w = np.asarray(weights, dtype=np.float64)
        if len(w) != m + 1:
            raise ValueError("one weight per replica (healthy replicas first, degraded last)")
        self.w = w
        smap = build_shard_map(k, plc.n1, plc.n2)
        self.h_cols = [smap.comp_columns(i) for i in range(plc.n1)]
        self.d_cols = [smap.sync_columns(j) for j in range(plc.n2)]
        # slots: healthy (r, i) -> r * n1 + i ; degraded j -> m * n1 + j
        self.n_slots = m * plc.n1 + plc.n2
        self.slot_elems = [len(self.h_cols[s % plc.n1]) * unit for s in range(m * plc.n1)] + \
                          [len(c) * unit for c in self.d_cols]
        self.slot_proc = [plc.hp[s // plc.n1][s % plc.n1] for s in range(m * plc.n1)] + list(plc.dp)
        self.hosted = [s for s in range(self.n_slots) if self.slot_proc[s] == self.rank]
        self.local = {s: self.ops.alloc(self.slot_elems[s] * self.eb) for s in self.hosted}
        self.sig = self.ops.alloc(SIG_BYTES)
        mine = {"slots": {s: self.ops.handle(p) for s, p in self.local.items()},
                "sig": self.ops.handle(self.sig)}
        table = [None] * self.world
        dist.all_gather_object(table, mine)
        # phase A/C plan on H_0's processes: unit j pairs H_0's copy with D's copy
        h_owner = np.empty(k, dtype=np.int64)
        h_off = np.empty(k, dtype=np.int64)
        d_owner = np.empty(k, dtype=np.int64)
        d_off = np.empty(k, dtype=np.int64)
        for i, c in enumerate(self.h_cols):
            h_owner[c], h_off[c] = i, np.arange(len(c)) * unit
        for j, c in enumerate(self.d_cols):
            d_owner[c], d_off[c] = m * plc.n1 + j, np.arange(len(c)) * unit
        mine_units = np.flatnonzero(np.asarray(plc.hp[0])[h_owner] == self.rank)
        self.plan = None
        self.slot_ptr = dict(self.local)
        self.opened = {}
        self.partners = set()
        if len(mine_units):
            for s in np.unique(d_owner[mine_units]).tolist():
                if s not in self.slot_ptr:
                    self.slot_ptr[s] = self.opened[s] = self.ops.open(table[self.slot_proc[s]]["slots"][s])
                if self.slot_proc[s] != self.rank:
                    self.partners.add(self.slot_proc[s])
            order = sorted(self.slot_ptr)
            idx = {s: n for n, s in enumerate(order)}
            self.bufs = [self.slot_ptr[s] for s in order]
            plan = Plan(dtype_code(dtype))
            plan.add_units(unit, [idx[int(s)] for s in h_owner[mine_units]], h_off[mine_units],
                           [idx[int(s)] for s in d_owner[mine_units]], d_off[mine_units])
            self.plan = plan.finalize()
        # degraded processes: partners are the H_0 processes that read/write them
        for j, p in enumerate(plc.dp):
            if p != self.rank:
                continue
            for i in np.unique(h_owner[self.d_cols[j]]).tolist():
                if plc.hp[0][i] != self.rank:
                    self.partners.add(plc.hp[0][i])
        self.partners = sorted(self.partners)
        self.peer_sig = {p: self.ops.open(table[p]["sig"]) for p in self.partners}
        self.is_h0 = any(plc.hp[0][i] == self.rank for i in range(plc.n1))
        self.is_d = self.rank in plc.dp
        # NCCL groups: healthy logical rank i across replicas (created by every rank, same order)
        self.groups = {}
        for i in range(plc.n1):
            procs = tuple(sorted({plc.hp[r][i] for r in range(m)}))
            if procs not in self.groups:
                self.groups[procs] = dist.new_group(list(procs)) if len(procs) > 1 else None
        self.epoch = 0
        self._status = None

    def upload(self) -> "NtpDpGroup":
        if self.plan is not None:
            self.plan.upload(self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        return self

    def arena(self, slot: int) -> torch.Tensor:
        return _wrap(self.local[slot], self.slot_elems[slot], self.dtype, self.device)

    def _words(self, kind, peers, mine: bool):
        if mine:  # words in my page written by `peers`
            return [self.sig + 8 * (kind * SIG_WORDS + p) for p in peers]
        return [self.peer_sig[p] + 8 * (kind * SIG_WORDS + self.rank) for p in peers]

    def step(self, stream=None, spin_ns: int = 20_000_000_000) -> None:
        L = _lib.load()
        self.epoch += 1
        e = self.epoch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        sp = ctypes.c_void_p(s.cuda_stream)
        st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        plc, m = self.plc, self.m
        if self.is_d and self.partners:
            _lib.check(L.ntp_signal_post(_lib.u64_ptr_array(self._words(READY, self.partners, False)),
                                         len(self.partners), e, sp), "ntp_signal_post")
        # A: fold D's contribution into H_0
        if self.plan is not None:
            if self.partners:
                w = self._words(READY, [p for p in self.partners], True)
                _lib.check(L.ntp_signal_wait(_lib.u64_ptr_array(w), len(w), e, spin_ns, st, sp),
                           "ntp_signal_wait")
            self.plan.grad_sync_into(self.bufs, OPS["weighted"], self.w[0], self.w[m], 1, s)
        # B: aligned all-reduce of the healthy replicas (pre-multiplied sums)
        with torch.cuda.stream(s):
            for i in range(plc.n1):
                procs = tuple(sorted({plc.hp[r][i] for r in range(m)}))
                mine = [r for r in range(m) if plc.hp[r][i] == self.rank]
                if not mine or len(procs) < 2:
                    continue
                r = mine[0]
                t = self.arena(r * plc.n1 + i)
                if t.element_size() >= 4:
                    # every rank uses the same NCCL op: pre-mul-sum, H_0's factor 1
                    op = dist._make_nccl_premul_sum(self._factor(1.0 if r == 0 else self.w[r], t))
                    dist.all_reduce(t, op=op, group=self.groups[procs])
                else:
                    # torch's 16-bit pre-mul-sum mis-scales (measured on B200); weight
                    # H_r (r > 0) in place with the uniform kernel, then a plain SUM
                    if r > 0:
                        w = (ctypes.c_double * 1)(float(self.w[r]))
                        _lib.check(L.ntp_uniform_sync(_lib.ptr_array([t.data_ptr()]), 1, t.numel(),
                                                      dtype_code(t.dtype), OPS["weighted"], w, sp),
                                   "ntp_uniform_sync")
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.groups[procs])
        # C: push the result into D's arena, then release D
        if self.plan is not None:
            self.plan.reshard(self.bufs, s)
            if self.partners:
                w = self._words(DONE, self.partners, False)
                _lib.check(L.ntp_signal_post(_lib.u64_ptr_array(w), len(w), e, sp), "ntp_signal_post")
        if self.is_d and self.partners:
            w = self._words(DONE, self.partners, True)
            _lib.check(L.ntp_signal_wait(_lib.u64_ptr_array(w), len(w), e, spin_ns, st, sp),
                       "ntp_signal_wait")

    def _factor(self, w: float, t: torch.Tensor) -> torch.Tensor:
        # torch's ProcessGroupNCCL takes an fp32 device scalar for 16-bit dtypes
        dt = torch.float64 if t.dtype == torch.float64 else torch.float32
        key = (float(w), dt)
        cache = self.__dict__.setdefault("_factors", {})
        if key not in cache:
            cache[key] = torch.tensor([float(w)], dtype=dt, device=t.device)
        return cache[key]

    def status(self) -> int:
        return int(self._status.item()) if self._status is not None else 0

    def close(self) -> None:
        """Collective: unmap peers' memory, wait until every process has, then free ours."""
        torch.cuda.synchronize(self.device)
        for p in list(self.opened.values()) + list(self.peer_sig.values()):
            self.ops.close(p)
        dist.barrier()
        for p in self.local.values():
            self.ops.free(p)
        self.ops.free(self.sig)
        self.opened, self.peer_sig, self.local = {}, {}, {}
