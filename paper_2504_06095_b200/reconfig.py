"""Reconfiguration on a failure event: redistribute weights and optimizer state
from one TP layout to another (north_star item 3).

The reference has no such function (no optimizer).  Its building
blocks are the ownership algebra -- ``build_reshard_plan`` / ``apply_plan``
(shardmap.py:185-217), ``contiguous_assignment`` (tpnumerics.py:115-120) and
the contiguous-interval planner ``naive_contiguous_sync_volumes``
(shardmap.py:220-245) -- and this module turns them into data movement:

* degraded replica: contiguous TP-n1 -> contiguous TP-n2 (its sync layout);
  units whose old owner died are sourced from a *backup* replica's copy (a
  healthy DP replica holds identical weights and optimizer state);
* healthy replicas: contiguous TP-n1 -> the NTP comp layout of the shard map
  (comp is contiguous only when n2 in {n1, 1}).

Every state tensor is a set of per-rank unit-major buffers; one plan moves all
units of one dtype with the ``ntp_reshard`` copy kernel (bit-exact).  Buffer
numbering inside a plan: source ranks, then destination ranks, then backup ranks.
"""

from __future__ import annotations

import numpy as np
import torch

from .plans import Plan, dtype_code, layout_offsets, tensor_ptrs
from .shardmap import ShardMap
from .tpnumerics import assignment_from_comp, assignment_from_sync, contiguous_assignment


def layouts_for_failure(k: int, n1: int, n2: int, smap: ShardMap | None = None):
    """(contiguous TP-n1, degraded TP-n2 sync layout, healthy NTP comp layout)."""
    from .shardmap import build_shard_map
    smap = smap if smap is not None else build_shard_map(k, n1, n2)
    return contiguous_assignment(k, n1), assignment_from_sync(smap), assignment_from_comp(smap)


def build_reconfig_plan(k: int, unit: int, src_cols, dst_cols, dtype, *, dead=(),
                        backup_cols=None, plan: Plan | None = None, src_base=None,
                        dst_base=None, backup_base=None) -> Plan:
    """Append a segment moving k units from layout src_cols to dst_cols.

    dead: source ranks whose memory is gone; their units come from backup_cols
    (the same columns in a surviving replica, buffers numbered after dst).
    """
    n_src, n_dst = len(src_cols), len(dst_cols)
    s_owner, s_off = layout_offsets(src_cols, k, unit, src_base)
    d_owner, d_off = layout_offsets(dst_cols, k, unit, dst_base)
    a_buf = s_owner.copy()
    a_off = s_off.copy()
    dead = set(int(d) for d in dead)
    if dead:
        if backup_cols is None:
            raise ValueError("units of a dead rank need a backup replica layout")
        b_owner, b_off = layout_offsets(backup_cols, k, unit, backup_base)
        lost = np.isin(s_owner, list(dead))
        a_buf[lost] = n_src + n_dst + b_owner[lost]
        a_off[lost] = b_off[lost]
    plan = Plan(dtype_code(dtype)) if plan is None else plan
    plan.add_units(unit, a_buf, a_off, n_src + d_owner, d_off)
    return plan


def reconfigure(src, dst, plan: Plan, backup=(), stream=None) -> None:
    """Run a finalized reconfiguration plan: dst[...] <- src / backup units.
    src, dst, backup: lists of per-rank device tensors (unit-major)."""
    tensors = list(src) + list(dst) + list(backup)
    if plan.device is None:
        plan.upload(tensors[0].device.index)
    plan.reshard(tensor_ptrs(tensors), stream)


def reconfigure_state(states: dict, k: int, unit: int, src_cols, dst_cols, *, dead=(),
                      backup_cols=None, backups: dict | None = None):
    """Move several state tensors (e.g. {"param": bf16, "master": fp32, "exp_avg": fp32,
    "exp_avg_sq": fp32}) from src_cols to dst_cols.  states[name] = (src_list, dst_list);
    backups[name] = backup rank list.  One plan per dtype is cached across names."""
    plans = {}
    for name, (src, dst) in states.items():
        dt = src[0].dtype
        if dt not in plans:
            plans[dt] = build_reconfig_plan(k, unit, src_cols, dst_cols, dt, dead=dead,
                                            backup_cols=backup_cols).finalize()
        bk = () if backups is None else backups.get(name, ())
        reconfigure(src, dst, plans[dt], bk)
    return plans


def ownership_after(src_owner: np.ndarray, dst_cols) -> np.ndarray:
    """Column -> rank ownership after the move (for replay checks with apply_plan)."""
    out = np.empty_like(src_owner)
    for r, cols in enumerate(dst_cols):
        out[np.asarray(cols)] = r
    return out


def alloc_layout(cols, unit: int, dtype, device) -> list[torch.Tensor]:
    """Zeroed per-rank unit-major buffers for a layout."""
    return [torch.zeros(len(c) * unit, dtype=dtype, device=device) for c in cols]
