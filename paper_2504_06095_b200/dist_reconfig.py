"""Reconfiguration on failure across processes (SURVEY 8(f) row 1 at N > 1).

One GPU of the degraded replica D has died.  Both DP replicas leave the
contiguous TP-n1 layout they trained in (``contiguous_assignment``,
tpnumerics.py:115-120):

* H (healthy): TP-n1 contiguous -> the NTP comp layout of ``build_shard_map``
  (shardmap.py:141-182);
* D (degraded): its n1-1 survivors -> TP-n2 contiguous (the sync layout);
  the dead rank's units are read from H's TP-n1 copy, which holds identical
  weights and optimizer state.

Every process *pulls* the units of the destination arenas it hosts: sources
on the same GPU are local reads, others are CUDA-IPC-mapped peer reads over
NVLink.  One ``ntp_reshard`` launch per state tensor (bit-exact copy kernel,
DESIGN.md 4), between two barriers: before it every source is complete, after
it no process may reuse a source that a peer still reads.

Global slot numbering: H_src i -> i, D_src i -> n1 + i, H_dst i -> 2 n1 + i,
D_dst j -> 3 n1 + j.  The survivors keep their GPUs: D_dst j is hosted where
D_src survivors[j] was.  Host logic runs on CPU under gloo with a fake
``DeviceOps`` (tests/test_dist_reconfig.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .dist import DeviceOps, _wrap
from .plans import Plan, dtype_code, layout_offsets
from .shardmap import build_shard_map
from .tpnumerics import assignment_from_comp, assignment_from_sync, contiguous_assignment


@dataclass(frozen=True)
class FailureLayout:
    """Per-segment layouts of a failure reconfiguration.  segs: (k, unit) of
    every partitioned tensor group (MLP columns of a layer, heads, ...)."""

    n1: int
    n2: int
    dead: int
    segs: tuple

    def survivors(self) -> list:
        return [r for r in range(self.n1) if r != self.dead]

    def n_slots(self) -> int:
        return 3 * self.n1 + self.n2

    def layouts(self, k: int):
        smap = build_shard_map(k, self.n1, self.n2)
        return contiguous_assignment(k, self.n1), assignment_from_comp(smap), \
            assignment_from_sync(smap)

    def slot_elems(self) -> list:
        """Elements of every slot's arena (all segments, unit-major)."""
        el = np.zeros(self.n_slots(), dtype=np.int64)
        for k, unit in self.segs:
            contig, comp, sync = self.layouts(k)
            for i in range(self.n1):
                el[i] += len(contig[i]) * unit
                el[self.n1 + i] += len(contig[i]) * unit
                el[2 * self.n1 + i] += len(comp[i]) * unit
            for j in range(self.n2):
                el[3 * self.n1 + j] += len(sync[j]) * unit
        if self.dead >= 0:
            el[self.n1 + self.dead] = 0  # that GPU's memory is gone
        return el.tolist()

    def units(self):
        """Per segment: (unit, src_slot, src_off, dst_slot, dst_off) over the
        segment's 2k destination units (H's k, then D's k), global slots."""
        if self.n1 - 1 != self.n2 and self.dead >= 0:
            raise ValueError(f"one dead rank takes TP{self.n1} to TP{self.n1 - 1}, not TP{self.n2}")
        base = np.zeros(self.n_slots(), dtype=np.int64)
        out = []
        for k, unit in self.segs:
            contig, comp, sync = self.layouts(k)
            n1 = self.n1
            s_own, s_off = layout_offsets(contig, k, unit, base[:n1])
            sd_own, sd_off = layout_offsets(contig, k, unit, base[n1:2 * n1])
            h_own, h_off = layout_offsets(comp, k, unit, base[2 * n1:3 * n1])
            d_own, d_off = layout_offsets(sync, k, unit, base[3 * n1:])
            # H: contiguous -> comp, all local to the replica
            a_slot = [s_own]
            a_off = [s_off]
            b_slot = [2 * n1 + h_own]
            b_off = [h_off]
            # D: survivors' contiguous copies -> sync; the dead rank's units from H
            src_slot = n1 + sd_own
            src_off = sd_off.copy()
            lost = sd_own == self.dead
            src_slot[lost] = s_own[lost]
            src_off[lost] = s_off[lost]
            a_slot.append(src_slot)
            a_off.append(src_off)
            b_slot.append(3 * n1 + d_own)
            b_off.append(d_off)
            out.append((unit, np.concatenate(a_slot), np.concatenate(a_off),
                        np.concatenate(b_slot), np.concatenate(b_off)))
            for i in range(n1):
                base[i] += len(contig[i]) * unit
                if i != self.dead:
                    base[n1 + i] += len(contig[i]) * unit
                base[2 * n1 + i] += len(comp[i]) * unit
            for j in range(self.n2):
                base[3 * n1 + j] += len(sync[j]) * unit
        return out


def failure_placement(n1: int, dead: int, world: int):
    """slot -> world rank for H_src/H_dst (first half of the GPUs), D_src/D_dst
    (second half).  world >= 2n1: one logical rank per GPU; smaller worlds pack
    logical ranks onto GPUs in proportion (like dist.Placement.default)."""
    if world >= 2 * n1:
        hp = list(range(n1))
        dp = list(range(n1, 2 * n1))
    elif world == 1:
        hp, dp = [0] * n1, [0] * n1
    else:
        gh = world // 2
        gd = world - gh
        hp = [i * gh // n1 for i in range(n1)]
        dp = [gh + i * gd // n1 for i in range(n1)]
    survivors = [r for r in range(n1) if r != dead]
    proc = hp + dp + hp + [dp[s] for s in survivors]
    return proc


class DistReconfig:
    """One process's share of a multi-GPU failure reconfiguration.

    states: {name: dtype}, e.g. {"param": bf16, "master": fp32, "exp_avg": fp32,
    "exp_avg_sq": fp32}.  Every hosted slot gets one arena per state name
    (``arena(slot, name)`` is a torch view); fill the H_src / D_src arenas,
    call ``run()``, read the H_dst / D_dst arenas."""

    def __init__(self, lay: FailureLayout, proc: list, states: dict, device: int,
                 ops: DeviceOps | None = None, group=None):
        self.lay, self.proc, self.states, self.device = lay, list(proc), dict(states), device
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ops = ops if ops is not None else DeviceOps(device)
        self.slot_elems = lay.slot_elems()
        dead_slot = lay.n1 + lay.dead if lay.dead >= 0 else -1
        self.hosted = [s for s in range(lay.n_slots()) if self.proc[s] == self.rank and s != dead_slot]
        self.local = {}
        for name, dt in self.states.items():
            eb = torch.empty(0, dtype=dt).element_size()
            for s in self.hosted:
                self.local[(s, name)] = self.ops.alloc(max(1, self.slot_elems[s]) * eb)
        mine = {"rank": self.rank,
                "slots": {f"{s}:{n}": self.ops.handle(p) for (s, n), p in self.local.items()}}
        table = [None] * self.world
        dist.all_gather_object(table, mine, group=group)
        # the units this process pulls: destinations it hosts
        units = []
        touched = set()
        for unit, a_slot, a_off, b_slot, b_off in lay.units():
            sel = np.flatnonzero(np.asarray([self.proc[int(b)] for b in b_slot]) == self.rank)
            if len(sel) == 0:
                continue
            units.append((unit, a_slot[sel], a_off[sel], b_slot[sel], b_off[sel]))
            touched.update(np.unique(a_slot[sel]).tolist())
            touched.update(np.unique(b_slot[sel]).tolist())
        if dead_slot in touched:
            raise RuntimeError("reconfiguration plan reads the dead rank")  # pragma: no cover
        self.units = sum(len(u[1]) for u in units)
        order = sorted(touched)
        self.buf_index = {s: i for i, s in enumerate(order)}
        self.opened = {}
        self.bufs = {}
        for name in self.states:
            ptrs = []
            for s in order:
                if (s, name) in self.local:
                    ptrs.append(self.local[(s, name)])
                else:
                    p = self.ops.open(table[self.proc[s]]["slots"][f"{s}:{name}"])
                    self.opened[(s, name)] = p
                    ptrs.append(p)
            self.bufs[name] = ptrs
        self.plans = {}
        self.split_plans = {}   # dt -> (local-source plan, peer-source plan)
        if units:
            remap = np.full(lay.n_slots(), -1, dtype=np.int64)
            for s, i in self.buf_index.items():
                remap[s] = i
            batches = self._interleave(units)
            local_src = self._is_local(remap)
            for dt in set(self.states.values()):
                plan = Plan(dtype_code(dt))
                for unit, a_s, a_o, b_s, b_o in batches:
                    plan.add_units(unit, remap[a_s], a_o, remap[b_s], b_o)
                self.plans[dt] = plan.finalize()
                parts = []
                for want_local in (True, False):
                    part = Plan(dtype_code(dt))
                    n = 0
                    for unit, a_s, a_o, b_s, b_o in batches:
                        sel = local_src[remap[a_s]] == want_local
                        if sel.any():
                            part.add_units(unit, remap[a_s][sel], a_o[sel], remap[b_s][sel], b_o[sel])
                            n += int(sel.sum())
                    parts.append(part.finalize() if n else None)
                self.split_plans[dt] = tuple(parts)
        # "interleaved" (default): one kernel per state tensor, local copies and
        # peer pulls interleaved in its chunk order; "split": two kernels on two
        # streams, the peer one capped to `peer_ctas` SMs -- measured no faster
        # (profiles/r01_dist_reconfig.json)
        self.launch_mode = "interleaved"
        self.peer_ctas = 40
        self._side = None

    def _interleave(self, units):
        """Order the pulled units so local copies (HBM-bound) and peer reads
        (NVLink-bound) are spread evenly through the plan: the kernel's CTAs
        then keep both in flight at once instead of running an HBM phase and a
        link phase back to back.  Key = the unit's byte-weighted position
        within its class; batches of one unit size feed Plan.add_units."""
        rows = []
        for unit, a_s, a_o, b_s, b_o in units:
            peer = np.asarray([self.proc[int(a)] != self.rank for a in a_s])
            rows.append((np.full(len(a_s), unit), a_s, a_o, b_s, b_o, peer))
        u = np.concatenate([r[0] for r in rows])
        a_s, a_o, b_s, b_o, peer = (np.concatenate([r[i] for r in rows]) for i in range(1, 6))
        key = np.empty(len(u), dtype=np.float64)
        for cls in (True, False):
            idx = np.flatnonzero(peer == cls)
            if len(idx):
                csum = np.cumsum(u[idx]).astype(np.float64)
                key[idx] = (csum - 0.5 * u[idx]) / csum[-1]
        order = np.argsort(key, kind="stable")
        u, a_s, a_o, b_s, b_o = u[order], a_s[order], a_o[order], b_s[order], b_o[order]
        cut = np.flatnonzero(np.diff(u)) + 1
        out = []
        for lo, hi in zip(np.r_[0, cut], np.r_[cut, len(u)]):
            out.append((int(u[lo]), a_s[lo:hi], a_o[lo:hi], b_s[lo:hi], b_o[lo:hi]))
        return out

    def _is_local(self, remap):
        """bool per dense buffer index: the buffer lives on this process."""
        order = sorted(self.buf_index, key=self.buf_index.get)
        return np.asarray([self.proc[s] == self.rank for s in order], dtype=bool)

    def upload(self) -> "DistReconfig":
        for p in self.plans.values():
            p.upload(self.device)
        for parts in self.split_plans.values():
            for p in parts:
                if p is not None:
                    p.upload(self.device)
        return self

    def arena(self, slot: int, name: str) -> torch.Tensor:
        return _wrap(self.local[(slot, name)], self.slot_elems[slot], self.states[name],
                     self.device)

    def run(self, stream=None) -> None:
        """Collective.  Pull every hosted destination unit (one reshard launch
        per state tensor), bracketed by barriers."""
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        self.launch(stream)
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)

    def launch(self, stream=None) -> None:
        """The copies alone (no barriers): the caller orders them."""
        if self.launch_mode != "split":
            for name, dt in self.states.items():
                if dt in self.plans:
                    self.plans[dt].reshard(self.bufs[name], stream)
            return
        from . import _lib
        L = _lib.load()
        main = torch.cuda.current_stream(self.device) if stream is None else stream
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        side = self._side
        side.wait_stream(main)
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        old_cap = int(L.ntp_get_option(1))
        try:
            for name, dt in self.states.items():
                if dt not in self.split_plans:
                    continue
                local, peer = self.split_plans[dt]
                if peer is not None:
                    L.ntp_set_option(1, self.peer_ctas)
                    peer.reshard(self.bufs[name], side)
                if local is not None:
                    L.ntp_set_option(1, max(1, sms - self.peer_ctas) if peer is not None else 0)
                    local.reshard(self.bufs[name], main)
        finally:
            L.ntp_set_option(1, old_cap)
        main.wait_stream(side)

    def bytes_pulled(self) -> dict:
        """Algorithmic bytes this process moves, split into local and over the link."""
        out = {"local": 0, "peer": 0}
        for name, dt in self.states.items():
            if dt not in self.plans:
                continue
            eb = torch.empty(0, dtype=dt).element_size()
            tab = self.plans[dt].export()
            order = sorted(self.buf_index, key=self.buf_index.get)
            for ab, _ao, _bb, _bo, ln in tab:
                key = "local" if self.proc[order[ab]] == self.rank else "peer"
                out[key] += int(ln) * eb
        return out

    def close(self) -> None:
        if torch.cuda.is_available():
            torch.cuda.synchronize(self.device)
        for p in self.opened.values():
            self.ops.close(p)
        self.opened = {}
        dist.barrier(group=self.group)
        for p in self.local.values():
            self.ops.free(p)
        self.local = {}
