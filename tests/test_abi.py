"""The C ABI: libntp_b200.so loads, exports every symbol include/ntp_b200.h
declares, and its host-side plan builder produces a chunk table that covers
every unit exactly once (no device calls: runs on CPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2504_06095_b200 import _lib
from paper_2504_06095_b200.plans import Plan
from paper_2504_06095_b200.shardmap import build_shard_map
from paper_2504_06095_b200.tpnumerics import (
    assignment_from_comp, assignment_from_sync, build_pair_plan,
)

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "ntp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntp_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = _lib.load()
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_library_is_sm100a():
    so = open(os.path.join(ROOT, "paper_2504_06095_b200", "libntp_b200.so"), "rb").read()
    assert b"sm_100a" in so


def test_errors_round_trip():
    L = _lib.load()
    comp = np.empty(8, dtype=np.int64)
    rc = L.ntp_shard_map(8, 4, 6, _lib.p64(comp), _lib.p64(comp))
    assert rc == _lib.NTP_EINVAL
    assert _lib.last_error() == "reduced degree n2=6 exceeds healthy degree n1=4"
    with pytest.raises(ValueError):
        _lib.check(rc)


def _coverage(plan, n_bufs, sizes):
    """Every element of every buffer is covered exactly once on side A and B."""
    tab = plan.export()
    cov = [np.zeros(s, dtype=np.int32) for s in sizes]
    for a_buf, a_off, b_buf, b_off, ln in tab:
        cov[a_buf][a_off:a_off + ln] += 1
        cov[b_buf][b_off:b_off + ln] += 1
    return cov, tab


@pytest.mark.parametrize("k,n1,n2,h", [(4096, 4, 3, 1024), (96, 8, 8, 4), (60, 6, 3, 8),
                                       (37, 16, 1, 3), (14336, 4, 2, 64)])
def test_pair_plan_covers_each_unit_once(k, n1, n2, h):
    smap = build_shard_map(k, n1, n2)
    hc, rc = assignment_from_comp(smap), assignment_from_sync(smap)
    plan = build_pair_plan(hc, rc, k, 2 * h, _lib.NTP_F32).finalize()
    st = plan.stats
    assert st["n_units"] == k and st["elems"] == k * 2 * h
    assert st["vectorized"] == (h % 2 == 0)
    sizes = [len(c) * 2 * h for c in hc] + [len(c) * 2 * h for c in rc]
    cov, tab = _coverage(plan, n1 + n2, sizes)
    for c in cov:
        assert (c == 1).all()
    # each chunk pairs the same column on both sides
    unit = 2 * h
    h_pos = {}
    for r, cols in enumerate(hc):
        for p, c in enumerate(cols):
            h_pos[(r, p)] = c
    r_pos = {}
    for r, cols in enumerate(rc):
        for p, c in enumerate(cols):
            r_pos[(n1 + r, p)] = c
    for a_buf, a_off, b_buf, b_off, ln in tab[:200]:
        assert h_pos[(a_buf, a_off // unit)] == r_pos[(b_buf, b_off // unit)]
        assert a_off % unit == b_off % unit


def test_runs_merge_for_contiguous_layouts():
    # n1 - n2 = 1: the offload rank's columns are contiguous per sync shard
    smap = build_shard_map(4096, 4, 3)
    plan = build_pair_plan(assignment_from_comp(smap), assignment_from_sync(smap), 4096, 2048,
                           _lib.NTP_F32).finalize()
    assert plan.stats["n_runs"] == 6  # kept prefix + offloaded tail per sync shard
    # n1 - n2 = 2: round-robin offload -> single-unit runs
    smap = build_shard_map(14336, 4, 2)
    plan = build_pair_plan(assignment_from_comp(smap), assignment_from_sync(smap), 14336, 128,
                           _lib.NTP_BF16).finalize()
    assert plan.stats["n_runs"] == 2 + 7168


def test_plan_state_errors():
    p = Plan(_lib.NTP_F32)
    with pytest.raises(RuntimeError):
        p.export()  # not finalized
    p.add_units(4, [0], [0], [1], [0]).finalize()
    with pytest.raises(RuntimeError):
        p.add_units(4, [0], [4], [1], [4])
    with pytest.raises(ValueError):
        Plan(_lib.NTP_F32).add_units(4, [70], [0], [1], [0])


def test_options_round_trip():
    L = _lib.load()
    assert L.ntp_get_option(0) == 0  # AUTO sync-kernel selection by default
    assert L.ntp_set_option(1, 24) == 0 and L.ntp_get_option(1) == 24
    assert L.ntp_set_option(1, 0) == 0 and L.ntp_get_option(1) == 0
    assert L.ntp_set_option(0, 9) == _lib.NTP_EINVAL
    assert L.ntp_set_option(7, 1) == _lib.NTP_EINVAL
    # NTP_OPT_PLAN_MIN_CHUNKS (default 1184 = 8 per SM) and NTP_OPT_SYNC_L2 (default 0)
    assert L.ntp_get_option(2) == 1184 and L.ntp_get_option(3) == 0
    assert L.ntp_set_option(2, 0) == 0 and L.ntp_get_option(2) == 0
    assert L.ntp_set_option(2, 1184) == 0
    assert L.ntp_set_option(3, 3) == _lib.NTP_EINVAL and L.ntp_set_option(2, -1) == _lib.NTP_EINVAL
    assert L.ntp_gemm_get_max_ctas() == 0


def test_min_chunks_splits_small_plans_alike_in_every_dtype():
    """Small plans get >= 1184 chunks; the chunk size is set in elements, so the
    same units split identically in bf16, fp32 and fp64."""
    import torch
    from paper_2504_06095_b200.workloads import ModelShape, build_plan, pair_layout
    lay = pair_layout(ModelShape("s", 1024, 1024, 0, 1), 4, 3)
    tabs = [build_plan(lay, dt).export() for dt in (torch.bfloat16, torch.float32, torch.float64)]
    assert len(tabs[0]) >= 1184
    assert all(np.array_equal(tabs[0], t) for t in tabs[1:])
