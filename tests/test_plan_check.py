"""Static memory-safety checks of every plan the product builds (CPU only).

compute-sanitizer is closed on the B200 pool, so out-of-bounds accesses and
write races of the plan-driven kernels are ruled out here instead: every
chunk of the plans the bench, the multi-GPU groups and the reconfiguration
build must lie inside its buffer, and no element may be written by two
chunks (two CTAs) of one launch (``ntp_plan_check``).  tests/test_bounds_gpu.py
adds device canaries around the buffers.
"""

import numpy as np
import pytest

from paper_2504_06095_b200 import _lib
from paper_2504_06095_b200.dist import Placement, process_plan_units
from paper_2504_06095_b200.plans import Plan
from paper_2504_06095_b200.reconfig import build_reconfig_plan, layouts_for_failure
from paper_2504_06095_b200.workloads import C1, GPT_1_3B, LLAMA3_8B, ModelShape, build_plan, pair_layout

BF16 = _lib.NTP_BF16


@pytest.mark.parametrize("shape,layers,n1,n2", [(GPT_1_3B, 24, 4, 3), (LLAMA3_8B, 2, 4, 3),
                                                (LLAMA3_8B, 1, 4, 2), (C1, 1, 4, 3),
                                                (ModelShape("odd", 36, 601, 6, 2), 2, 5, 2)])
def test_bench_plans_in_bounds_and_race_free(shape, layers, n1, n2):
    import torch
    lay = pair_layout(shape, n1, n2, layers=layers)
    plan = build_plan(lay, torch.bfloat16)
    plan.check(list(lay.h_elems) + list(lay.r_elems), write_sides=3)


@pytest.mark.parametrize("world", [2, 4, 7, 8])
@pytest.mark.parametrize("policy", ["split", "healthy"])
def test_per_process_plans_in_bounds_and_race_free(world, policy):
    """The plans each process of an N-GPU NtpSyncGroup runs (local + peer
    buffers): in bounds per buffer, and no element written twice across ALL
    processes' plans together (two GPUs never write the same unit)."""
    lay = pair_layout(GPT_1_3B, 4, 3, layers=2)
    plc = Placement.default(world, 4, 3)
    elems = list(lay.h_elems) + list(lay.r_elems)
    union = Plan(BF16)
    for rank in range(world):
        units, touched = process_plan_units(lay, plc, rank, policy)
        if not units:
            continue
        order = sorted(touched)
        remap = np.full(len(elems), -1, dtype=np.int64)
        remap[order] = np.arange(len(order))
        p = Plan(BF16)
        for unit, hs, ho, rs, ro in units:
            p.add_units(unit, remap[hs], ho, remap[rs], ro)
            union.add_units(unit, hs, ho, rs, ro)
        p.finalize().check([elems[s] for s in order], write_sides=3)
    union.finalize().check(elems, write_sides=3)


@pytest.mark.parametrize("k,n1,n2,dead", [(14336, 4, 3, 3), (4096, 4, 2, 1), (1000, 2, 1, 0)])
def test_reconfig_plans_in_bounds_and_race_free(k, n1, n2, dead):
    unit = 2 * 64
    contig, sync, comp = layouts_for_failure(k, n1, n2)
    import torch
    plan = build_reconfig_plan(k, unit, contig, sync, torch.bfloat16, dead=(dead,),
                               backup_cols=contig).finalize()
    sizes = ([len(c) * unit for c in contig] + [len(c) * unit for c in sync]
             + [len(c) * unit for c in contig])
    plan.check(sizes, write_sides=2)
    plan2 = build_reconfig_plan(k, unit, contig, comp, torch.bfloat16).finalize()
    plan2.check([len(c) * unit for c in contig] + [len(c) * unit for c in comp], write_sides=2)


def test_check_reports_out_of_bounds_and_overlap():
    p = Plan(BF16).add_units(64, [0, 0], [0, 64], [1, 1], [0, 64]).finalize()
    p.check([128, 128])
    with pytest.raises(ValueError, match="exceed its 100"):
        p.check([128, 100])
    with pytest.raises(ValueError, match="uses buffer 1 of 1"):
        p.check([128])
    q = Plan(BF16).add_units(64, [0, 0], [0, 32], [1, 1], [0, 64]).finalize()  # A ranges overlap
    with pytest.raises(ValueError, match="write overlapping elements of buffer 0"):
        q.check([128, 128], write_sides=3)
    q.check([128, 128], write_sides=2)  # side A only read: a copy plan may share sources
