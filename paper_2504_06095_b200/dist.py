"""Multi-GPU NTP gradient sync: one process per GPU, peer memory over NVSwitch.

Placement: the healthy TP-n1 replica's logical ranks and the degraded TP-n2
replica's logical ranks are hosted by world ranks (processes, one GPU each);
a process may host several logical ranks (e.g. N=2: the whole healthy
replica on GPU 0, the reduced one on GPU 1).

Data path (one-sided *push* from the reduced side):
  * every logical rank's gradient arena is a cudaMalloc'd buffer exported with
    CUDA IPC; each reduced-hosting process maps the healthy arenas it pairs
    with (its sync shards' comp owners, shardmap.py:160-180);
  * per step, healthy processes post a "ready" epoch into the reduced
    processes' signal pages; each reduced process runs ONE kernel that waits
    for its ready words, reads both copies of every unit of its sync shard (the
    healthy copy over NVLink), reduces w_h*g_h + w_r*g_r in fp32, writes the
    result to its own arena and into the healthy owner's arena (peer stores),
    and finally posts "done" to the healthy processes;
  * healthy processes block their stream on the done words.
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
from .tpnumerics import build_pair_plan
from .workloads import PairLayout

SIG_WORDS = 64             # per page: ready[64] then done[64] (uint64), slot = writer's world rank
SIG_BYTES = 2 * SIG_WORDS * 8
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


def process_plan_units(lay: PairLayout, plc: Placement, rank: int):
    """The units `rank` computes (those whose reduced owner it hosts), as
    per-segment (k, unit, cols, h_slot, h_off, r_slot, r_off) arrays in global
    slot numbering, plus the set of peer slots it touches."""
    out = []
    touched = set()
    my_red = {j for j, p in enumerate(plc.r_proc) if p == rank}
    for k, unit, hc, rc, hb, rb in lay.segs:
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
        sel = np.flatnonzero(np.isin(r_owner, list(my_red)))
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


def signal_wiring(lay: PairLayout, plc: Placement, rank: int):
    """(ready_from, done_to, done_from): world ranks this process waits on for
    'ready', posts 'done' to (as a reduced host), and waits on for 'done' (as a
    healthy host).  Same-process pairs need no signal."""
    pairs = exchange_pairs(lay, plc)
    ready_from = sorted({h for h, r in pairs if r == rank and h != rank})
    done_to = ready_from
    done_from = sorted({r for h, r in pairs if h == rank and r != rank})
    return ready_from, done_to, done_from


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
                 ops: DeviceOps | None = None, group=None):
        self.lay, self.plc, self.dtype = lay, placement, dtype
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
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
        # 3. what this process computes, and which peer buffers it needs
        units, touched = process_plan_units(lay, placement, self.rank)
        self.ready_from, self.done_to, self.done_from = signal_wiring(lay, placement, self.rank)
        self.opened = {}
        self.slot_ptr = dict(self.local)
        for s in sorted(touched):
            if s not in self.slot_ptr:
                proc = placement.proc_of_slot(s)
                self.slot_ptr[s] = self.opened[s] = self.ops.open(table[proc]["slots"][s])
        self.peer_sig = {}
        for p in set(self.done_to) | set(self.done_from) | set(self.ready_from):
            self.peer_sig[p] = self.ops.open(table[p]["sig"])
        # 4. the plan, with buffers renumbered to a dense local table
        order = sorted(self.slot_ptr)
        self.buf_index = {s: i for i, s in enumerate(order)}
        self.bufs = [self.slot_ptr[s] for s in order]
        self.plan = None
        if units:
            remap = np.full(placement.n1 + placement.n2, -1, dtype=np.int64)
            for s, i in self.buf_index.items():
                remap[s] = i
            plan = Plan(dtype_code(dtype))
            for unit, hs, ho, rs, ro in units:
                plan.add_units(unit, remap[hs], ho, remap[rs], ro)
            self.plan = plan.finalize()
        self.units = sum(len(u[1]) for u in units)
        # signal words: where I wait / where I post
        self.wait_ready = [self.sig + 8 * (READY * SIG_WORDS + p) for p in self.ready_from]
        self.post_done = [self.peer_sig[p] + 8 * (DONE * SIG_WORDS + self.rank) for p in self.done_to]
        self.post_ready = [self.peer_sig[p] + 8 * (READY * SIG_WORDS + self.rank)
                           for p in self.done_from]
        self.wait_done = [self.sig + 8 * (DONE * SIG_WORDS + p) for p in self.done_from]
        self.epoch = 0
        self._status = None

    # -- device-side -----------------------------------------------------------

    def upload(self) -> "NtpSyncGroup":
        if self.plan is not None:
            self.plan.upload(self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        return self

    def arena(self, slot: int) -> torch.Tensor:
        """Torch view of a hosted logical rank's gradient arena."""
        return _wrap(self.local[slot], self.slot_elems[slot], self.dtype, self.device)

    def step(self, w_h: float, w_r: float, stream=None, spin_ns: int = 20_000_000_000) -> None:
        """One synchronisation; stream-ordered on `stream` (default: current)."""
        L = _lib.load()
        self.epoch += 1
        e = self.epoch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        sp = ctypes.c_void_p(s.cuda_stream)
        st = ctypes.cast(self._status.data_ptr(), ctypes.POINTER(ctypes.c_int))
        if self.post_ready:
            _lib.check(L.ntp_signal_post(_lib.u64_ptr_array(self.post_ready), len(self.post_ready),
                                         e, sp), "ntp_signal_post")
        if self.plan is not None:
            if self.wait_ready or self.post_done:
                self.plan.grad_sync_signaled(self.bufs, OPS["weighted"], w_h, w_r,
                                             self.wait_ready, self.post_done, e, spin_ns,
                                             self._status.data_ptr(), s)
            else:
                self.plan.grad_sync(self.bufs, OPS["weighted"], w_h, w_r, s)
        if self.wait_done:
            _lib.check(L.ntp_signal_wait(_lib.u64_ptr_array(self.wait_done), len(self.wait_done),
                                         e, spin_ns, st, sp), "ntp_signal_wait")

    def status(self) -> int:
        return int(self._status.item()) if self._status is not None else 0

    def close(self) -> None:
        for p in list(self.opened.values()) + list(self.peer_sig.values()):
            self.ops.close(p)
        self.opened, self.peer_sig = {}, {}
        for p in self.local.values():
            self.ops.free(p)
        self.ops.free(self.sig)
        self.local = {}


def aligned_all_reduce(tensor: torch.Tensor, weight: float | None = None, group=None) -> None:
    """NCCL fall-through for naturally aligned shards (uniform_grad_sync,
    tpnumerics.py:263-286, across processes): SUM, or per-rank weighted sum via
    NCCL's pre-multiplied-sum op (each rank scales its own input inside NCCL --
    no separate scale kernel)."""
    if weight is None or weight == 1.0:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
        return
    op = dist._make_nccl_premul_sum(float(weight))
    dist.all_reduce(tensor, op=op, group=group)
