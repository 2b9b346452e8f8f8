"""DP > 2 with one degraded replica across processes (BASELINE configs[2]:
DP=4 x TP2 with one replica degraded to TP1, batch-proportional weights).

Replicas: m healthy TP-n1 replicas H_0..H_{m-1}, identically laid out (the NTP
comp layout of (k, n1, n2), shardmap.py:141-182), and one degraded TP-n2
replica D (the sync layout).  Every unit must end as

    v = sum_r w_r * g_r        (H replicas and D, replica order H_0.., D)

in all m+1 owners.  The healthy replicas are aligned with each other, so
their part is an NCCL all-reduce; only the exchange with D is nonuniform.
Every healthy arena is cut into pieces, and each piece into m sub-ranges;
replica r owns the r-th sub-range of every piece (the fold and push-back work
is spread over all healthy GPUs).  Per step, per piece p, on every healthy
process:

  A  its sub-range: g_r <- w_r * g_r + w_D * g_D, D's copy read over NVLink
     (ntp_grad_sync_ex, write A only); the rest of the piece: g_r <- w_r * g_r
  B  NCCL SUM of the piece across the healthy replicas (second stream)
  C  its sub-range's result pushed into D's arena (ntp_reshard over peer
     memory, third stream)

so B(p) overlaps A(p+1) and C(p-1); then "done" goes to D, whose stream waits
for every partner's.

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
from .dist import READY, DONE, SIG_BYTES, SIG_WORDS, DeviceOps, _wrap, check_signal_world
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
                 device: int, weights, ops: DeviceOps | None = None, pieces: int = 1):
        """pieces > 1 pipelines the step: every healthy arena is cut into
        `pieces` unit ranges, and piece p's fold-in (A), NCCL all-reduce (B) and
        push-back (C) run on three streams, so B(p) overlaps A(p+1) and C(p-1)."""
        if pieces < 1:
            raise ValueError("pieces must be >= 1")
        self.k, self.unit, self.m, self.plc, self.dtype = k, unit, m, plc, dtype
        self.device = device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        check_signal_world(self.world)
        self.ops = ops if ops is not None else DeviceOps(device)
        self.eb = torch.empty(0, dtype=dtype).element_size()
        w = np.asarray(weights, dtype=np.float64)
        if len(w) != m + 1:
            raise ValueError("one weight per replica (healthy replicas first, degraded last)")
        self.w = w
        n1 = plc.n1
        smap = build_shard_map(k, n1, plc.n2)
        self.h_cols = [smap.comp_columns(i) for i in range(n1)]
        self.d_cols = [smap.sync_columns(j) for j in range(plc.n2)]
        # slots: healthy (r, i) -> r * n1 + i ; degraded j -> m * n1 + j
        self.n_slots = m * n1 + plc.n2
        self.slot_elems = [len(self.h_cols[s % n1]) * unit for s in range(m * n1)] + \
                          [len(c) * unit for c in self.d_cols]
        self.slot_proc = [plc.hp[s // n1][s % n1] for s in range(m * n1)] + list(plc.dp)
        self.hosted = [s for s in range(self.n_slots) if self.slot_proc[s] == self.rank]
        reps = {s // n1 for s in self.hosted if s < m * n1}
        if len(reps) > 1:
            raise ValueError("a process may host logical ranks of one healthy replica only")
        self.replica = reps.pop() if reps else None
        self.local = {s: self.ops.alloc(self.slot_elems[s] * self.eb) for s in self.hosted}
        self.sig = self.ops.alloc(SIG_BYTES)
        mine = {"slots": {s: self.ops.handle(p) for s, p in self.local.items()},
                "sig": self.ops.handle(self.sig)}
        table = [None] * self.world
        dist.all_gather_object(table, mine)
        # where every unit lives in D: unit j -> (slot, offset)
        d_slot = np.empty(k, dtype=np.int64)
        d_off = np.empty(k, dtype=np.int64)
        for j, c in enumerate(self.d_cols):
            d_slot[c], d_off[c] = m * n1 + j, np.arange(len(c)) * unit
        # Pieces cut every healthy logical rank's arena into position ranges;
        # inside a piece, replica r folds D into (and later pushes back) the
        # r-th of m sub-ranges, so every healthy GPU shares the link work.
        self.pieces = pieces
        self.bounds = [np.linspace(0, len(c), pieces + 1).astype(np.int64) for c in self.h_cols]
        self.fold = [[] for _ in range(pieces)]    # (slot, pos_lo, pos_hi) folded here
        self.scale = [[] for _ in range(pieces)]   # (slot, pos_lo, pos_hi) only scaled here
        self.partners = set()
        touched = set()
        for slot in self.hosted:
            if slot >= m * n1:
                continue
            r, i = divmod(slot, n1)
            for pc in range(pieces):
                lo, hi = int(self.bounds[i][pc]), int(self.bounds[i][pc + 1])
                a = lo + (hi - lo) * r // m
                b = lo + (hi - lo) * (r + 1) // m
                if b > a:
                    self.fold[pc].append((slot, a, b))
                    ds = d_slot[self.h_cols[i][a:b]]
                    touched.update(np.unique(ds).tolist())
                for x, y in ((lo, a), (b, hi)):
                    if y > x:
                        self.scale[pc].append((slot, x, y))
        self.slot_ptr = dict(self.local)
        self.opened = {}
        for ds in sorted(touched):
            if ds not in self.slot_ptr:
                self.slot_ptr[ds] = self.opened[ds] = self.ops.open(table[self.slot_proc[ds]]["slots"][ds])
            if self.slot_proc[ds] != self.rank:
                self.partners.add(self.slot_proc[ds])
        order = sorted(self.slot_ptr)
        idx = {s: n for n, s in enumerate(order)}
        self.bufs = [self.slot_ptr[s] for s in order]
        self.plans = [None] * pieces        # fold (A, weighted) and push-back (C, copy)
        self.scale_plans = [None] * pieces  # scale-only units: x <- w_r * x
        for pc in range(pieces):
            if self.fold[pc]:
                plan = Plan(dtype_code(dtype))
                for slot, a, b in self.fold[pc]:
                    cols = self.h_cols[slot % n1][a:b]
                    plan.add_units(unit, np.full(b - a, idx[slot]), np.arange(a, b) * unit,
                                   [idx[int(x)] for x in d_slot[cols]], d_off[cols])
                self.plans[pc] = plan.finalize()
            if self.scale[pc]:
                plan = Plan(dtype_code(dtype))
                for slot, a, b in self.scale[pc]:
                    pos = np.arange(a, b) * unit
                    plan.add_units(unit, np.full(b - a, idx[slot]), pos, np.full(b - a, idx[slot]), pos)
                self.scale_plans[pc] = plan.finalize()
        self.plan = next((p for p in self.plans if p is not None), None)
        # degraded processes: partners are the healthy processes that fold its units
        my_d = {m * n1 + j for j, p in enumerate(plc.dp) if p == self.rank}
        if my_d:
            for r in range(m):
                for i in range(n1):
                    for pc in range(pieces):
                        lo, hi = int(self.bounds[i][pc]), int(self.bounds[i][pc + 1])
                        a, b = lo + (hi - lo) * r // m, lo + (hi - lo) * (r + 1) // m
                        if b > a and my_d & set(np.unique(d_slot[self.h_cols[i][a:b]]).tolist()):
                            if plc.hp[r][i] != self.rank:
                                self.partners.add(plc.hp[r][i])
        self.partners = sorted(self.partners)
        self.peer_sig = {p: self.ops.open(table[p]["sig"]) for p in self.partners}
        self.is_h = self.replica is not None
        self.is_d = self.rank in plc.dp
        # NCCL groups: healthy logical rank i across replicas (created by every rank, same order)
        self.groups = {}
        for i in range(n1):
            procs = tuple(sorted({plc.hp[r][i] for r in range(m)}))
            if procs not in self.groups:
                self.groups[procs] = dist.new_group(list(procs)) if len(procs) > 1 else None
        self.epoch = 0
        self._status = None

    def upload(self) -> "NtpDpGroup":
        for p in self.plans + self.scale_plans:
            if p is not None:
                p.upload(self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        self._streams = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))
        return self

    def arena(self, slot: int) -> torch.Tensor:
        return _wrap(self.local[slot], self.slot_elems[slot], self.dtype, self.device)

    def _words(self, kind, peers, mine: bool):
        if mine:  # words in my page written by `peers`
            return [self.sig + 8 * (kind * SIG_WORDS + p) for p in peers]
        return [self.peer_sig[p] + 8 * (kind * SIG_WORDS + self.rank) for p in peers]

    def step(self, stream=None, spin_ns: int = 20_000_000_000) -> None:
        """One sync.  D posts ready; every healthy process, per piece:
        A  g_r <- w_r * g_r + w_D * g_D on its fold sub-range (D's copy read
           over NVLink), g_r <- w_r * g_r on the rest of the piece;
        B  NCCL SUM of the piece across the healthy replicas (own stream);
        C  its fold sub-range's result pushed into D's arena (third stream);
        then posts done to D, whose stream waits for every partner's done."""
        L = _lib.load()
        self.epoch += 1
        e = self.epoch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        sp = ctypes.c_void_p(s.cuda_stream)
        st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        m = self.m
        if self.is_d and self.partners:
            _lib.check(L.ntp_signal_post(_lib.u64_ptr_array(self._words(READY, self.partners, False)),
                                         len(self.partners), e, sp), "ntp_signal_post")
        if self.is_h and self.partners:
            w = self._words(READY, self.partners, True)
            _lib.check(L.ntp_signal_wait(_lib.u64_ptr_array(w), len(w), e, spin_ns, st, sp),
                       "ntp_signal_wait")
        sB, sC = self._streams
        if self.is_h:
            w_r = float(self.w[self.replica])
            for pc in range(self.pieces):
                if self.plans[pc] is not None:
                    self.plans[pc].grad_sync_into(self.bufs, OPS["weighted"], w_r,
                                                  float(self.w[m]), 1, s)
                if self.scale_plans[pc] is not None:
                    self.scale_plans[pc].grad_sync_into(self.bufs, OPS["weighted"], w_r, 0.0, 1, s)
                sB.wait_stream(s)
                with torch.cuda.stream(sB):
                    self._all_reduce_piece(pc)
                if self.plans[pc] is not None:
                    sC.wait_stream(sB)
                    self.plans[pc].reshard(self.bufs, sC)
            s.wait_stream(sB)
            s.wait_stream(sC)
            if self.partners:
                w = self._words(DONE, self.partners, False)
                _lib.check(L.ntp_signal_post(_lib.u64_ptr_array(w), len(w), e, sp), "ntp_signal_post")
        if self.is_d and self.partners:
            w = self._words(DONE, self.partners, True)
            _lib.check(L.ntp_signal_wait(_lib.u64_ptr_array(w), len(w), e, spin_ns, st, sp),
                       "ntp_signal_wait")

    def _all_reduce_piece(self, pc: int) -> None:
        """Phase B for one piece on the current stream: every hosted healthy
        logical rank's (already weighted) arena range, summed across the
        healthy replicas by NCCL."""
        plc, m = self.plc, self.m
        for i in range(plc.n1):
            procs = tuple(sorted({plc.hp[r][i] for r in range(m)}))
            slot = None if self.replica is None else self.replica * plc.n1 + i
            if slot not in self.local or len(procs) < 2:
                continue
            lo, hi = (int(b) * self.unit for b in self.bounds[i][pc:pc + 2])
            if hi > lo:
                dist.all_reduce(self.arena(slot)[lo:hi], op=dist.ReduceOp.SUM,
                                group=self.groups[procs])

    def status(self) -> int:
        return int(self._status.item()) if self._status is not None else 0

    def close(self) -> None:
        """Collective: unmap peers' memory, wait until every process has, then free ours."""
        if torch.cuda.is_available():
            torch.cuda.synchronize(self.device)
        for p in list(self.opened.values()) + list(self.peer_sig.values()):
            self.ops.close(p)
        dist.barrier()
        for p in self.local.values():
            self.ops.free(p)
        self.ops.free(self.sig)
        self.opened, self.peer_sig, self.local = {}, {}, {}


def balanced_executors(proc: np.ndarray, iters: int = 64) -> np.ndarray:
    """Pick, for every unit (column of proc [R x k] = the process holding each
    of its R copies), the process that reads all copies and writes them back.

    Per direction a process moves (R-1) unit copies for every unit it executes
    and one for every other unit it holds, i.e. load_p = held_p + (R-2) * E_p.
    Units with the same owner tuple form a group; executions are moved inside
    each group from its most to its least loaded owner until the maximum load
    stops falling (water-filling), then every group hands out contiguous runs
    of its columns to its owners.  A GPU that already holds more units (the
    degraded replica) executes fewer of them."""
    R, k = proc.shape
    held = {}
    for p in proc.ravel().tolist():
        held[p] = held.get(p, 0) + 1
    keys, inv = np.unique(proc.T, axis=0, return_inverse=True)
    inv = inv.ravel()
    sizes = np.bincount(inv, minlength=len(keys))
    owners = [sorted(set(row.tolist())) for row in keys]
    E = [{o: 0.0 for o in ow} for ow in owners]
    for gi, ow in enumerate(owners):          # start: equal shares
        for o in ow:
            E[gi][o] = sizes[gi] / len(ow)

    def load():
        out = dict.fromkeys(held, 0.0)
        for p in held:
            out[p] = float(held[p])
        for gi in range(len(owners)):
            for o, e in E[gi].items():
                out[o] += (R - 2) * e
        return out

    for _ in range(iters):
        ld = load()
        moved = False
        for gi, ow in enumerate(owners):
            if len(ow) < 2:
                continue
            hi = max(ow, key=lambda o: ld[o] if E[gi][o] > 0 else -1)
            lo = min(ow, key=lambda o: ld[o])
            gap = ld[hi] - ld[lo]
            if gap <= 1e-9 or E[gi][hi] <= 0 or R <= 2:
                continue
            step = min(E[gi][hi], gap / (2 * (R - 2)))
            E[gi][hi] -= step
            E[gi][lo] += step
            ld[hi] -= (R - 2) * step
            ld[lo] += (R - 2) * step
            moved = True
        if not moved:
            break
    ex = np.empty(k, dtype=np.int64)
    for gi, ow in enumerate(owners):
        cols = np.flatnonzero(inv == gi)
        counts = np.floor([E[gi][o] for o in ow]).astype(np.int64)
        counts[-1] = len(cols) - counts[:-1].sum()   # exact total, remainder to the last
        if counts[-1] < 0:                            # pragma: no cover - rounding guard
            counts = np.full(len(ow), len(cols) // len(ow))
            counts[-1] = len(cols) - counts[:-1].sum()
        ex[cols] = np.repeat(np.asarray(ow, dtype=np.int64), counts)
    return ex


class NtpDpMultiGroup:
    """DP > 2 in one kernel per process (no NCCL): every unit has R = m + 1
    copies (m healthy replicas in the comp layout, the degraded one in the sync
    layout), and exactly one process -- one of the unit's owners -- reads all R
    copies over NVLink / HBM, forms sum_r w_r * g_r, and writes it to all R
    (ntp_multi_sync with peer-mapped buffers).  Executors are balanced by
    ``balanced_executors``; when every replica sits on its own GPU that is
    2 (R-1)/R * S * b bytes per GPU and direction -- what a ring all-reduce of
    a uniform DP group moves -- with no separate fold-in / push-back around it.  Ordering: ready
    to every partner, wait for theirs, one kernel, done, wait for theirs."""

    def __init__(self, k: int, unit: int, m: int, plc: DpPlacement, dtype: torch.dtype,
                 device: int, weights, ops: DeviceOps | None = None):
        from .plans import MultiPlan
        self.k, self.unit, self.m, self.plc, self.dtype = k, unit, m, plc, dtype
        self.device = device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        check_signal_world(self.world)
        self.ops = ops if ops is not None else DeviceOps(device)
        self.eb = torch.empty(0, dtype=dtype).element_size()
        R = m + 1
        w = np.asarray(weights, dtype=np.float64)
        if len(w) != R:
            raise ValueError("one weight per replica (healthy replicas first, degraded last)")
        self.w = w
        n1 = plc.n1
        smap = build_shard_map(k, n1, plc.n2)
        self.h_cols = [smap.comp_columns(i) for i in range(n1)]
        self.d_cols = [smap.sync_columns(j) for j in range(plc.n2)]
        self.n_slots = m * n1 + plc.n2
        self.slot_elems = [len(self.h_cols[s % n1]) * unit for s in range(m * n1)] + \
                          [len(c) * unit for c in self.d_cols]
        self.slot_proc = [plc.hp[s // n1][s % n1] for s in range(m * n1)] + list(plc.dp)
        self.hosted = [s for s in range(self.n_slots) if self.slot_proc[s] == self.rank]
        self.local = {s: self.ops.alloc(self.slot_elems[s] * self.eb) for s in self.hosted}
        self.sig = self.ops.alloc(SIG_BYTES)
        mine = {"slots": {s: self.ops.handle(p) for s, p in self.local.items()},
                "sig": self.ops.handle(self.sig)}
        table = [None] * self.world
        dist.all_gather_object(table, mine)
        # copies of every unit: slot[r][u], off[r][u] (r < m healthy, r = m degraded)
        slot = np.empty((R, k), dtype=np.int64)
        off = np.empty((R, k), dtype=np.int64)
        for i, c in enumerate(self.h_cols):
            for r in range(m):
                slot[r, c], off[r, c] = r * n1 + i, np.arange(len(c)) * unit
        for j, c in enumerate(self.d_cols):
            slot[m, c], off[m, c] = m * n1 + j, np.arange(len(c)) * unit
        proc = np.asarray(self.slot_proc)[slot]                 # [R, k]
        ex_proc = balanced_executors(proc)
        mine_u = np.flatnonzero(ex_proc == self.rank)
        # partners: owners of my executed units' copies, and executors of units I own
        partners = set(np.unique(proc[:, mine_u]).tolist())
        owns = np.any(proc == self.rank, axis=0)
        partners |= set(np.unique(ex_proc[owns]).tolist())
        partners.discard(self.rank)
        self.partners = sorted(partners)
        self.slot_ptr = dict(self.local)
        self.opened = {}
        for s in sorted(set(np.unique(slot[:, mine_u]).tolist())):
            if s not in self.slot_ptr:
                self.slot_ptr[s] = self.opened[s] = self.ops.open(table[self.slot_proc[s]]["slots"][s])
        order = sorted(self.slot_ptr)
        idx = np.full(self.n_slots, -1, dtype=np.int64)
        for n, s in enumerate(order):
            idx[s] = n
        self.bufs = [self.slot_ptr[s] for s in order]
        self.plan = None
        self.units = len(mine_u)
        if len(mine_u):
            self.plan = MultiPlan(dtype_code(dtype), R).add_units(
                unit, idx[slot[:, mine_u]], off[:, mine_u]).finalize()
        self.peer_sig = {p: self.ops.open(table[p]["sig"]) for p in self.partners}
        self.epoch = 0
        self._status = None

    def upload(self) -> "NtpDpMultiGroup":
        if self.plan is not None:
            self.plan.upload(self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        return self

    def arena(self, slot: int) -> torch.Tensor:
        return _wrap(self.local[slot], self.slot_elems[slot], self.dtype, self.device)

    def _words(self, kind, mine: bool):
        if mine:
            return [self.sig + 8 * (kind * SIG_WORDS + p) for p in self.partners]
        return [self.peer_sig[p] + 8 * (kind * SIG_WORDS + self.rank) for p in self.partners]

    def step(self, stream=None, spin_ns: int = 20_000_000_000) -> None:
        L = _lib.load()
        self.epoch += 1
        e = self.epoch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        sp = ctypes.c_void_p(s.cuda_stream)
        st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        n = len(self.partners)
        none = _lib.u64_ptr_array([])

        def exchange(kind):
            # post this process's words and wait for the partners' in one launch
            # (ntp_grad_sync_step with no plan runs only the handshakes)
            _lib.check(L.ntp_grad_sync_step(
                None, None, 0, OPS["weighted"], 1.0, 1.0,
                _lib.u64_ptr_array(self._words(kind, False)), n,
                _lib.u64_ptr_array(self._words(kind, True)), n, none, 0, none, 0,
                e, int(spin_ns), st, sp), "ntp_grad_sync_step")

        if n:
            exchange(READY)
        if self.plan is not None:
            self.plan.sync(self.bufs, OPS["weighted"], self.w, s)
        if n:
            exchange(DONE)

    def status(self) -> int:
        return int(self._status.item()) if self._status is not None else 0

    def close(self) -> None:
        if torch.cuda.is_available():
            torch.cuda.synchronize(self.device)
        for p in list(self.opened.values()) + list(self.peer_sig.values()):
            self.ops.close(p)
        dist.barrier()
        for p in self.local.values():
            self.ops.free(p)
        self.ops.free(self.sig)
        self.opened, self.peer_sig, self.local = {}, {}, {}
