"""Multi-GPU NTP gradient sync: one process per GPU, peer memory over NVSwitch.

Placement: the healthy TP-n1 replica's logical ranks and the degraded TP-n2
replica's logical ranks are hosted by world ranks (processes, one GPU each);
a process may host several logical ranks (e.g. N=2: the whole healthy
replica on GPU 0, the reduced one on GPU 1).

Data path (one-sided pulls + pushes over peer memory):
  * every logical rank's gradient arena is a cudaMalloc'd buffer exported with
    CUDA IPC; each process maps the arenas of the processes it shares units
    with (a reduced rank's sync shard pairs with its comp owners,
    shardmap.py:160-180);
  * every unit is computed by exactly one of its two owners' GPUs: for each
    (healthy GPU, reduced GPU) pair the units are split in half, so both GPUs
    read the partner's copy and write the result into both copies at once
    (``unit_executors``); the busiest GPU's link bytes per direction stay at
    the lower bound S_g*b;
  * per step every process posts a "ready" epoch into its partners' signal
    pages, runs ONE kernel that waits for its partners' ready words, reduces
    w_h*g_h + w_r*g_r in fp32 for its units, writes both copies (local and peer
    stores) and, once all its CTAs' stores have landed, posts "done"; the
    stream then blocks on the partners' done words.
This is the reference's pre-sync reshard + pairwise reduce + post-sync
reshard (tpnumerics.py:323-356) as a single kernel with no staging buffer and
no intermediate collective.  Regions whose layouts align (n1 == n2, or
healthy<->healthy replicas) fall through to NCCL all-reduce
(``aligned_all_reduce``).

Host logic (placement, plan per process, signal wiring, handle exchange) is
kept free of device calls behind ``DeviceOps`` so it runs under gloo on CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .plans import OPS, Plan, dtype_code
from .workloads import PairLayout

SIG_WORDS = 64             # per page: ready[64] then done[64] (uint64), slot = writer's world rank
SIG_BYTES = 2 * SIG_WORDS * 8


def check_signal_world(world: int) -> None:
    """Signal slots are indexed by the writer's world rank inside a page of
    SIG_WORDS ready words then SIG_WORDS done words: a larger world would
    alias ready onto done words (or write past the page)."""
    if world > SIG_WORDS:
        raise ValueError(f"signal page holds {SIG_WORDS} ranks, world size is {world}")
READY, DONE = 0, 1


@dataclass(frozen=True)
class Placement:
    """World rank hosting each logical rank of the healthy and reduced replicas."""

    n1: int
    n2: int
    h_proc: tuple
    r_proc: tuple

    @classmethod
    def default(cls, world: int, n1: int, n2: int) -> "Placement":
        if world >= n1 + n2:       # one logical rank per GPU; spare GPUs idle ("failed")
            return cls(n1, n2, tuple(range(n1)), tuple(range(n1, n1 + n2)))
        if world == 1:
            return cls(n1, n2, (0,) * n1, (0,) * n2)
        # split the GPUs between the replicas in proportion to their degrees
        gh = max(1, min(world - 1, round(world * n1 / (n1 + n2))))
        gr = world - gh
        h = tuple(i * gh // n1 for i in range(n1))
        r = tuple(gh + i * gr // n2 for i in range(n2))
        return cls(n1, n2, h, r)

    def hosted(self, rank: int):
        """Buffer slots hosted by `rank`: healthy logical i -> slot i, reduced j -> n1 + j."""
        return [i for i, p in enumerate(self.h_proc) if p == rank] + \
               [self.n1 + j for j, p in enumerate(self.r_proc) if p == rank]

    def proc_of_slot(self, slot: int) -> int:
        return self.h_proc[slot] if slot < self.n1 else self.r_proc[slot - self.n1]


def unit_executors(lay: PairLayout, plc: Placement, policy: str = "split", seg_filter=None):
    """Per segment: (h_owner, h_off, r_owner, r_off, executor_proc) arrays over
    the k units.  Units whose two owners share a process run there.  Otherwise
    ``policy`` decides which endpoint computes the unit:

    * "split" (default): for every (healthy proc, reduced proc) pair, the first
      half of the pair's units (in column order) run on the reduced side and
      the second half on the healthy side -- both GPUs read and write over the
      link at once (measured: ~700 GB/s per direction vs ~495 GB/s when one
      side both reads and writes everything, profiles/r01_nvlink_probe.json);
    * "reduced": every unit runs on its reduced owner's GPU (pure push);
    * "healthy": every unit runs on its healthy owner's GPU -- the degraded
      GPU, which already serves twice the units, does no sync work at all;
    * a number x in [0, 1]: that share of each pair's units on the reduced side.
    """
    out = []
    hp_of = np.asarray(plc.h_proc)
    rp_of = np.asarray(plc.r_proc)
    for si, (k, unit, hc, rc, hb, rb) in enumerate(lay.segs):
        if seg_filter is not None and not seg_filter(si):
            continue
        h_owner = np.empty(k, dtype=np.int64)
        h_off = np.empty(k, dtype=np.int64)
        r_owner = np.empty(k, dtype=np.int64)
        r_off = np.empty(k, dtype=np.int64)
        for r, c in enumerate(hc):
            h_owner[c] = r
            h_off[c] = hb[r] + np.arange(len(c)) * unit
        for r, c in enumerate(rc):
            r_owner[c] = r
            r_off[c] = rb[r] + np.arange(len(c)) * unit
        hp, rp = hp_of[h_owner], rp_of[r_owner]
        ex = rp.copy()
        share = reduced_share(policy)
        if share < 1.0:
            key = hp * (1 << 20) + rp
            for kv in np.unique(key[hp != rp]):
                idx = np.flatnonzero(key == kv)
                ex[idx[int(np.ceil(len(idx) * share)):]] = hp[idx[0]]
        out.append((unit, h_owner, h_off, r_owner, r_off, ex))
    return out


def reduced_share(policy) -> float:
    """Share of each (healthy GPU, reduced GPU) pair's units computed on the
    reduced side under an executor policy."""
    named = {"split": 0.5, "reduced": 1.0, "healthy": 0.0}
    if policy in named:
        return named[policy]
    try:
        x = float(policy)
    except (TypeError, ValueError):
        raise ValueError(f"unknown executor policy {policy!r}") from None
    if not 0.0 <= x <= 1.0:
        raise ValueError(f"executor share must be in [0, 1], got {x}")
    return x


def process_plan_units(lay: PairLayout, plc: Placement, rank: int, policy: str = "split",
                       seg_filter=None):
    """The units `rank` computes, as per-segment (unit, h_slot, h_off, r_slot,
    r_off) arrays in global slot numbering, plus the set of slots it touches.
    seg_filter(i): restrict to some segments (a pipelined piece)."""
    out = []
    touched = set()
    for unit, h_owner, h_off, r_owner, r_off, ex in unit_executors(lay, plc, policy, seg_filter):
        sel = np.flatnonzero(ex == rank)
        if len(sel) == 0:
            continue
        out.append((unit, h_owner[sel], h_off[sel], plc.n1 + r_owner[sel], r_off[sel]))
        touched.update(np.unique(h_owner[sel]).tolist())
        touched.update((plc.n1 + np.unique(r_owner[sel])).tolist())
    return out, touched


def exchange_pairs(lay: PairLayout, plc: Placement) -> set:
    """(healthy proc, reduced proc) pairs that share at least one unit: reduced
    logical j pairs with the comp owners of its sync shard (its own kept prefix
    and the offload ranks holding its offloaded columns, shardmap.py:165-180)."""
    pairs = set()
    for k, unit, hc, rc, hb, rb in lay.segs:
        comp = np.empty(k, dtype=np.int64)
        for r, c in enumerate(hc):
            comp[c] = r
        for j, c in enumerate(rc):
            for i in np.unique(comp[c]):
                pairs.add((plc.h_proc[int(i)], plc.r_proc[j]))
    return pairs


def partners(lay: PairLayout, plc: Placement, rank: int) -> list:
    """World ranks this process exchanges units with (either direction).  Every
    step, a process posts "ready" to each partner, runs its kernel (which waits
    for the partners' "ready" and posts "done" to them when all its stores have
    landed) and then waits for each partner's "done"."""
    pairs = exchange_pairs(lay, plc)
    return sorted({r for h, r in pairs if h == rank and r != rank} |
                  {h for h, r in pairs if r == rank and h != rank})


class DeviceOps:
    """The device side of the group (replaced by a fake in CPU tests)."""

    def __init__(self, device: int):
        self.device = device
        self.L = _lib.load()

    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _lib.check(self.L.ntp_alloc(self.device, int(nbytes), ctypes.byref(p)), "ntp_alloc")
        return int(p.value)

    def handle(self, ptr: int) -> bytes:
        buf = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        _lib.check(self.L.ntp_ipc_get_handle(ctypes.c_void_p(ptr), buf), "ntp_ipc_get_handle")
        return buf.raw

    def open(self, handle: bytes) -> int:
        p = ctypes.c_void_p()
        _lib.check(self.L.ntp_ipc_open(self.device, handle, ctypes.byref(p)), "ntp_ipc_open")
        return int(p.value)

    def close(self, ptr: int) -> None:
        self.L.ntp_ipc_close(ctypes.c_void_p(ptr))

    def free(self, ptr: int) -> None:
        self.L.ntp_free(ctypes.c_void_p(ptr))


def _wrap(ptr: int, numel: int, dtype: torch.dtype, device: int) -> torch.Tensor:
    """A torch view of a raw device allocation (through __cuda_array_interface__)."""
    nbytes = numel * torch.empty(0, dtype=dtype).element_size()

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}

    with torch.cuda.device(device):
        t = torch.as_tensor(_CAI(), device=f"cuda:{device}")
    return t.view(dtype)


class NtpSyncGroup:
    """One process's share of a distributed nonuniform gradient sync."""

    def __init__(self, lay: PairLayout, placement: Placement, dtype: torch.dtype, device: int,
                 ops: DeviceOps | None = None, group=None, policy: str = "split",
                 pieces=None, aligned: str = "peer", prescaled: bool = False):
        """pieces: optional list of segment-index lists.  Each piece gets its
        own plan, so a caller can sync piece i as soon as its gradients (or its
        host-to-device copies) are in place: ``step(..., piece=i)``.  Every
        process must step the pieces in the same order (epochs pair up).

        aligned: with n1 == n2 the two replicas' shards line up (comp layout ==
        sync layout, identical arenas per rank pair); "nccl" then syncs each
        healthy/reduced arena pair with an NCCL all-reduce (aligned_all_reduce,
        the fall-through of uniform_grad_sync, tpnumerics.py:263-286) instead
        of the peer-memory kernel; "peer" (default, measured faster on B200:
        DESIGN.md 5) keeps the kernel.  Ignored when n1 != n2.

        prescaled (aligned="nccl" only): the gradients already carry their
        replica's batch weight (folded into the wgrad GEMM's alpha, e.g.
        MlpShard.backward(alpha=w)), so step() runs a plain NCCL SUM with no
        weighting pass; step()'s weights are then ignored."""
        if aligned not in ("peer", "nccl"):
            raise ValueError(f"aligned must be 'peer' or 'nccl', got {aligned!r}")
        self.pieces = [sorted(int(i) for i in p) for p in pieces] if pieces else []
        for p in self.pieces:
            if not p or p != list(range(p[0], p[-1] + 1)):
                raise ValueError("a piece must be a non-empty contiguous range of segments")
        self.lay, self.plc, self.dtype, self.policy = lay, placement, dtype, policy
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        check_signal_world(self.world)
        self.device = device
        self.ops = ops if ops is not None else DeviceOps(device)
        self.eb = torch.empty(0, dtype=dtype).element_size()
        elems = list(lay.h_elems) + list(lay.r_elems)
        self.slot_elems = elems
        self.hosted = placement.hosted(self.rank)
        # 1. local arenas + signal page
        self.local = {s: self.ops.alloc(elems[s] * self.eb) for s in self.hosted}
        self.sig = self.ops.alloc(SIG_BYTES)
        # 2. exchange IPC handles (objects travel over the host group: gloo or nccl)
        mine = {"rank": self.rank, "slots": {s: self.ops.handle(p) for s, p in self.local.items()},
                "sig": self.ops.handle(self.sig)}
        table = [None] * self.world
        dist.all_gather_object(table, mine, group=group)
        self.table = table
        # 3. which partners this process hand-shakes with, then its plans
        self.partners = partners(lay, placement, self.rank)
        self.opened = {}
        self.slot_ptr = dict(self.local)
        self.peer_sig = {p: self.ops.open(table[p]["sig"]) for p in self.partners}
        self.plan = None
        self.piece_plans = []
        self._build_plans(policy)
        # signal words (slot = writer's world rank in the receiver's page)
        self.post_ready = [self.peer_sig[p] + 8 * (READY * SIG_WORDS + self.rank)
                           for p in self.partners]
        self.wait_ready = [self.sig + 8 * (READY * SIG_WORDS + p) for p in self.partners]
        self.post_done = [self.peer_sig[p] + 8 * (DONE * SIG_WORDS + self.rank)
                          for p in self.partners]
        self.wait_done = [self.sig + 8 * (DONE * SIG_WORDS + p) for p in self.partners]
        self.epoch = 0
        self._status = None
        # True: step() is one launch (ntp_grad_sync_step), 25 -> 17.5 us at 1 MB
        # per replica, but 6 of 66 sweep measurements came out 15-60 % slow
        # (cause not found; profiles/r01_sweep_sync_multi.json).  False (default):
        # three launches (post ready / signalled sync / wait done), no outliers
        # in the same runs, and no difference at the bench's 2.4 GB.
        self.fused_step = False
        # CUDA-graph steps only: two launches (ready post, then the sync kernel
        # whose last CTA posts done and waits for the partners' done)
        self.two_launch = False
        self._sig_arrays = None
        self._bufs_array = None
        self.aligned = aligned if lay.n1 == lay.n2 else "peer"
        self.prescaled = bool(prescaled) and self.aligned == "nccl"
        self._aligned_pairs = self._aligned_groups(group) if self.aligned == "nccl" else None

    def _build_plans(self, policy) -> None:
        """What this process computes under an executor policy, which peer
        buffers it needs (IPC-mapped on first use), and the plans over a dense
        local buffer table (whole layout + one per piece)."""
        lay, placement = self.lay, self.plc
        units, touched = process_plan_units(lay, placement, self.rank, policy)
        for s in sorted(touched):
            if s not in self.slot_ptr:
                proc = placement.proc_of_slot(s)
                self.slot_ptr[s] = self.opened[s] = self.ops.open(self.table[proc]["slots"][s])
        order = sorted(self.slot_ptr)
        self.buf_index = {s: i for i, s in enumerate(order)}
        self.bufs = [self.slot_ptr[s] for s in order]
        self._bufs_array = None
        remap = np.full(placement.n1 + placement.n2, -1, dtype=np.int64)
        for s, i in self.buf_index.items():
            remap[s] = i
        self.plan = None
        if units:
            plan = Plan(dtype_code(self.dtype))
            for unit, hs, ho, rs, ro in units:
                plan.add_units(unit, remap[hs], ho, remap[rs], ro)
            self.plan = plan.finalize()
        self.units = sum(len(u[1]) for u in units)
        self.piece_plans = []
        for seg_ids in self.pieces:
            sel = set(seg_ids)
            pu, ptouched = process_plan_units(lay, placement, self.rank, policy,
                                              seg_filter=sel.__contains__)
            if not pu:
                self.piece_plans.append(None)
                continue
            if not ptouched <= set(self.buf_index):
                raise RuntimeError("piece touches a slot the whole plan does not")  # pragma: no cover
            pp = Plan(dtype_code(self.dtype))
            for unit, hs, ho, rs, ro in pu:
                pp.add_units(unit, remap[hs], ho, remap[rs], ro)
            self.piece_plans.append(pp.finalize())
        self.policy = policy

    def _aligned_groups(self, group):
        """(healthy slot, reduced slot, 2-process NCCL group or None when both
        slots live in this process) for every aligned pair this process hosts.
        new_group is collective: every process creates every pair's group, in
        ascending pair order."""
        n1, plc = self.lay.n1, self.plc
        ranks = dist.get_process_group_ranks(group) if group is not None else list(range(self.world))
        groups = {}
        for i in range(n1):
            p, q = plc.proc_of_slot(i), plc.proc_of_slot(i + n1)
            key = (min(p, q), max(p, q))
            if p != q and key not in groups:
                groups[key] = dist.new_group([ranks[key[0]], ranks[key[1]]])
        pairs = []
        for i in range(n1):
            p, q = plc.proc_of_slot(i), plc.proc_of_slot(i + n1)
            if self.rank in (p, q):
                pairs.append((i, i + n1, None if p == q else groups[(min(p, q), max(p, q))]))
        return pairs

    def _step_aligned(self, w_h: float, w_r: float, stream, piece) -> None:
        """n1 == n2 with aligned="nccl": per rank pair, one NCCL all-reduce of the
        (piece's range of the) two identical arenas, each side pre-weighted."""
        n1 = self.lay.n1
        with torch.cuda.stream(stream):
            for hs, rs, grp in self._aligned_pairs:
                rng = self.piece_ranges(piece) if piece is not None else None
                if grp is None:  # both copies in this process: one local 2-way kernel
                    a, b = self.arena(hs), self.arena(rs)
                    if rng is not None:
                        a, b = a[slice(*rng[hs])], b[slice(*rng[rs])]
                    L = _lib.load()
                    w = (ctypes.c_double * 2)(*((1.0, 1.0) if self.prescaled
                                                else (float(w_h), float(w_r))))
                    _lib.check(L.ntp_uniform_sync(_lib.ptr_array([a.data_ptr(), b.data_ptr()]), 2,
                                                  a.numel(), dtype_code(a.dtype), OPS["weighted"],
                                                  w, ctypes.c_void_p(stream.cuda_stream)),
                               "ntp_uniform_sync")
                    continue
                slot = hs if hs in self.local else rs
                t = self.arena(slot)
                if rng is not None:
                    t = t[slice(*rng[slot])]
                aligned_all_reduce(t, None if self.prescaled else (w_h if slot < n1 else w_r),
                                   group=grp)

    def set_policy(self, policy) -> "NtpSyncGroup":
        """Rebuild the plans for another executor policy (same arenas, same
        partners and signals); uploads them if the group was uploaded."""
        reduced_share(policy)  # validate before touching anything
        self._build_plans(policy)
        if self._status is not None:
            self.upload()
        return self

    # -- device-side -----------------------------------------------------------

    def upload(self) -> "NtpSyncGroup":
        if self.plan is not None:
            self.plan.upload(self.device)
        for pp in self.piece_plans:
            if pp is not None:
                pp.upload(self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        # device-resident epoch word (completed steps) for graph-replayed steps
        self._epoch_word = torch.zeros(1, dtype=torch.int64, device=f"cuda:{self.device}")
        self._word_epoch = 0   # the value the word holds once queued work has run
        self._graphs = {}
        return self

    def arena(self, slot: int) -> torch.Tensor:
        """Torch view of a hosted logical rank's gradient arena."""
        return _wrap(self.local[slot], self.slot_elems[slot], self.dtype, self.device)

    def piece_ranges(self, piece: int) -> dict:
        """slot -> (lo, hi) element range of a hosted arena that piece `piece`
        reads and writes (segments are contiguous in every arena)."""
        seg_ids = sorted(self.pieces[piece])
        out = {}
        for slot in self.hosted:
            side, idx = (0, slot) if slot < self.plc.n1 else (1, slot - self.plc.n1)
            first, last = self.lay.segs[seg_ids[0]], self.lay.segs[seg_ids[-1]]
            lo = int(first[4 + side][idx])
            hi = int(last[4 + side][idx]) + len(last[2 + side][idx]) * last[1]
            out[slot] = (lo, hi)
        return out

    def step(self, w_h: float, w_r: float, stream=None, spin_ns: int = 20_000_000_000,
             piece: int | None = None) -> None:
        """One synchronisation (of the whole layout, or of one piece); stream-
        ordered on `stream` (default: current)."""
        L = _lib.load()
        plan = self.plan if piece is None else self.piece_plans[piece]
        self.epoch += 1
        e = self.epoch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        if self.aligned == "nccl":
            self._step_aligned(w_h, w_r, s, piece)
            return
        sp = ctypes.c_void_p(s.cuda_stream)
        st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        if self._sig_arrays is None:  # ctypes arrays built once (host cost per step)
            self._sig_arrays = tuple(_lib.u64_ptr_array(w) for w in
                                     (self.post_ready, self.wait_ready, self.post_done,
                                      self.wait_done))
        pr, wr, pd, wd = self._sig_arrays
        if self._bufs_array is None:
            self._bufs_array = _lib.ptr_array(self.bufs)
        bufs = self._bufs_array
        if self.fused_step and self.partners:
            # one launch: post ready, wait ready, sync, post done, wait done
            _lib.check(L.ntp_grad_sync_step(
                plan._h if plan is not None else None, bufs, len(self.bufs), OPS["weighted"],
                float(w_h), float(w_r), pr, len(self.post_ready), wr, len(self.wait_ready),
                pd, len(self.post_done), wd, len(self.wait_done), e, int(spin_ns), st, sp),
                "ntp_grad_sync_step")
            return
        if self.post_ready:
            _lib.check(L.ntp_signal_post(pr, len(self.post_ready), e, sp), "ntp_signal_post")
        if plan is not None:
            if self.partners:
                _lib.check(L.ntp_grad_sync_signaled(
                    plan._h, bufs, len(self.bufs), OPS["weighted"], float(w_h), float(w_r),
                    wr, len(self.wait_ready), pd, len(self.post_done), e, int(spin_ns), st, sp),
                    "ntp_grad_sync_signaled")
            else:
                plan.grad_sync(self.bufs, OPS["weighted"], w_h, w_r, s)
        elif self.partners:
            # nothing to compute: wait until partners may be touched, then release them
            _lib.check(L.ntp_signal_wait(wr, len(self.wait_ready), e, spin_ns, st, sp),
                       "ntp_signal_wait")
            _lib.check(L.ntp_signal_post(pd, len(self.post_done), e, sp), "ntp_signal_post")
        if self.wait_done:
            _lib.check(L.ntp_signal_wait(wd, len(self.wait_done), e, spin_ns, st, sp),
                       "ntp_signal_wait")

    # -- CUDA-graph steps ------------------------------------------------------

    def _launch_dev(self, w_h: float, w_r: float, s, piece) -> None:
        """The step's launches with device-resident epochs (what step_graph
        records): the same kernels and handshakes as step(), each reading its
        epoch from the group's epoch word; the step's last launch advances it."""
        L = _lib.load()
        plan = self.plan if piece is None else self.piece_plans[piece]
        sp = ctypes.c_void_p(s.cuda_stream)
        st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        ew = ctypes.c_void_p(self._epoch_word.data_ptr())
        if self._sig_arrays is None:
            self._sig_arrays = tuple(_lib.u64_ptr_array(w) for w in
                                     (self.post_ready, self.wait_ready, self.post_done,
                                      self.wait_done))
        pr, wr, pd, wd = self._sig_arrays
        if self._bufs_array is None:
            self._bufs_array = _lib.ptr_array(self.bufs)
        bufs, spin = self._bufs_array, int(self._spin_ns)
        if not self.partners:
            if plan is not None:
                plan.grad_sync(self.bufs, OPS["weighted"], w_h, w_r, s)
            return
        if self.fused_step or self.two_launch:
            # two_launch: the ready post is its own (early) launch and the sync
            # kernel's last CTA posts done and waits for the partners' done
            if self.two_launch and not self.fused_step and self.post_ready:
                _lib.check(L.ntp_signal_post_dev(pr, len(self.post_ready), ew, sp),
                           "ntp_signal_post_dev")
            n_pre = len(self.post_ready) if self.fused_step else 0
            _lib.check(L.ntp_grad_sync_step_dev(
                plan._h if plan is not None else None, bufs, len(self.bufs), OPS["weighted"],
                float(w_h), float(w_r), pr, n_pre, wr, len(self.wait_ready),
                pd, len(self.post_done), wd, len(self.wait_done), ew, spin, st, sp),
                "ntp_grad_sync_step_dev")
            return
        if self.post_ready:
            _lib.check(L.ntp_signal_post_dev(pr, len(self.post_ready), ew, sp), "ntp_signal_post_dev")
        if plan is not None:
            _lib.check(L.ntp_grad_sync_signaled_dev(
                plan._h, bufs, len(self.bufs), OPS["weighted"], float(w_h), float(w_r),
                wr, len(self.wait_ready), pd, len(self.post_done), ew, spin, st, sp),
                "ntp_grad_sync_signaled_dev")
        else:
            _lib.check(L.ntp_signal_wait_dev(wr, len(self.wait_ready), ew, 0, spin, st, sp),
                       "ntp_signal_wait_dev")
            _lib.check(L.ntp_signal_post_dev(pd, len(self.post_done), ew, sp), "ntp_signal_post_dev")
        _lib.check(L.ntp_signal_wait_dev(wd, len(self.wait_done), ew, 1, spin, st, sp),
                   "ntp_signal_wait_dev")

    _spin_ns = 20_000_000_000

    def step_graph(self, w_h: float, w_r: float, stream=None, piece: int | None = None,
                   steps: int = 1, prologue=None) -> None:
        """`steps` synchronisations as ONE CUDA-graph launch (recorded on first
        use for this (piece, weights, steps, launch variant), replayed after):
        the host cost of a step drops to one graph launch, and on the device
        the step's kernels run back to back.  Same kernels, signals and
        results as step(); each process must issue the same sequence of steps
        (graph or not) so that epochs pair up.  prologue: optional callable
        recorded before each step (e.g. a benchmark's L2 flush).  Recording a new
        graph synchronizes the device once (torch.cuda.graph); replays do not.
        The graphs hold the group's plans: set_policy()/upload() drop them."""
        if self.aligned == "nccl":
            for _ in range(steps):
                self.step(w_h, w_r, stream, piece=piece)
            return
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        plan = self.plan if piece is None else self.piece_plans[piece]
        if plan is None and not self.partners and prologue is None:
            self.epoch += steps  # nothing to run here (e.g. the idle GPU at N=8)
            return
        key = (piece, float(w_h), float(w_r), int(steps), bool(self.fused_step),
               bool(self.two_launch), prologue)
        g = self._graphs.get(key)
        if g is None:
            if len(self._graphs) >= 16:  # e.g. a caller passing a new prologue each time
                self._graphs.clear()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.device)
            cap.wait_stream(s)
            with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                for _ in range(steps):
                    if prologue is not None:
                        prologue()
                    self._launch_dev(w_h, w_r, cap, piece)
            s.wait_stream(cap)
            self._graphs[key] = g
        if self._word_epoch != self.epoch:  # eager steps ran since: re-base the word
            with torch.cuda.stream(s):
                self._epoch_word.fill_(self.epoch)
            self._word_epoch = self.epoch
        with torch.cuda.stream(s):
            g.replay()
        self.epoch += steps
        self._word_epoch = self.epoch

    def open_slots(self, slots) -> list:
        """Device pointers of the given logical slots (IPC-mapping peers' arenas
        on first use): the partner copies a fused wgrad+sync GEMM reduces into."""
        out = []
        for s in slots:
            if s not in self.slot_ptr:
                proc = self.plc.proc_of_slot(s)
                self.slot_ptr[s] = self.opened[s] = self.ops.open(self.table[proc]["slots"][s])
            out.append(self.slot_ptr[s])
        return out

    def signal(self, kind: str, epoch: int, stream=None, spin_ns: int = 20_000_000_000) -> None:
        """Stream-ordered handshake with every partner: kind = "post_ready",
        "wait_ready", "post_done" or "wait_done" (the words step() uses)."""
        if not self.partners:
            return
        L = _lib.load()
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        sp = ctypes.c_void_p(s.cuda_stream)
        words = {"post_ready": self.post_ready, "wait_ready": self.wait_ready,
                 "post_done": self.post_done, "wait_done": self.wait_done}[kind]
        arr = _lib.u64_ptr_array(words)
        if kind.startswith("post"):
            _lib.check(L.ntp_signal_post(arr, len(words), int(epoch), sp), "ntp_signal_post")
        else:
            st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
            _lib.check(L.ntp_signal_wait(arr, len(words), int(epoch), spin_ns, st, sp),
                       "ntp_signal_wait")

    def status(self) -> int:
        return int(self._status.item()) if self._status is not None else 0

    def close(self) -> None:
        """Collective: unmap peers' memory, wait until every process has, then free ours."""
        if torch.cuda.is_available():
            torch.cuda.synchronize(self.device)
        for p in list(self.opened.values()) + list(self.peer_sig.values()):
            self.ops.close(p)
        self.opened, self.peer_sig = {}, {}
        dist.barrier()
        for p in self.local.values():
            self.ops.free(p)
        self.ops.free(self.sig)
        self.local = {}
        self._graphs = {}
        # the aligned pairs' NCCL groups stay with the default group, which
        # destroy_process_group() tears down with every subgroup


def aligned_all_reduce(tensor: torch.Tensor, weight: float | None = None, group=None) -> None:
    """NCCL fall-through for naturally aligned shards (uniform_grad_sync,
    tpnumerics.py:263-286, across processes): SUM, or per-rank weighted sum via
    NCCL's pre-multiplied-sum op (each rank scales its own input inside NCCL --
    no separate scale kernel).  Every rank of the group must pass a weight, or
    none (NCCL requires one op across the group).  16-bit tensors: torch's
    pre-mul-sum mis-scales them (measured on B200), so the weight is applied in
    place by ntp_uniform_sync before a plain SUM."""
    if weight is None:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
        return
    if tensor.element_size() < 4:
        w = (ctypes.c_double * 1)(float(weight))
        stream = torch.cuda.current_stream(tensor.device)
        _lib.check(_lib.load().ntp_uniform_sync(_lib.ptr_array([tensor.data_ptr()]), 1,
                                                tensor.numel(), dtype_code(tensor.dtype),
                                                OPS["weighted"], w,
                                                ctypes.c_void_p(stream.cuda_stream)),
                   "ntp_uniform_sync")
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
        return
    fdt = torch.float64 if tensor.dtype == torch.float64 else torch.float32
    factor = torch.tensor([float(weight)], dtype=fdt, device=tensor.device)
    dist.all_reduce(tensor, op=dist._make_nccl_premul_sum(factor), group=group)
