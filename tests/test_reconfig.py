"""Reconfiguration on failure (paper_2504_06095_b200/reconfig.py): TP-n1 ->
TP-n2 moves of weights / optimizer state.  CPU: the plan's chunk table,
replayed on numpy, equals the oracle's permutation copy and the ownership
replay of build_reshard_plan/apply_plan.  GPU: the ntp_reshard kernel is
bit-exact with the oracle for bf16 and fp32 state tensors."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2504_06095_b200.reconfig import (
    build_reconfig_plan, layouts_for_failure, ownership_after,
)
from paper_2504_06095_b200.shardmap import (
    POST_SYNC, PRE_SYNC, apply_plan, build_reshard_plan, build_shard_map,
)


def _positions(cols, k):
    owner = np.empty(k, dtype=np.int64)
    pos = np.empty(k, dtype=np.int64)
    for r, c in enumerate(cols):
        owner[c] = r
        pos[c] = np.arange(len(c))
    return owner, pos


def _oracle_move(src_bufs, dst_shapes, src_cols, dst_cols, k, unit, dead=(), backup=None,
                 backup_cols=None):
    s_owner, s_pos = _positions(src_cols, k)
    d_owner, d_pos = _positions(dst_cols, k)
    srcs = list(src_bufs)
    src_buf = s_owner.copy()
    src_pos = s_pos.copy()
    if dead:
        b_owner, b_pos = _positions(backup_cols, k)
        lost = np.isin(s_owner, list(dead))
        src_buf[lost] = len(srcs) + b_owner[lost]
        src_pos[lost] = b_pos[lost]
        srcs += list(backup)
    dst = [np.zeros(n, dtype=src_bufs[0].dtype) for n in dst_shapes]
    O.reshard_copy(srcs, dst, unit, src_buf, src_pos, d_owner, d_pos)
    return dst


def _replay(plan, bufs):
    for ab, ao, bb, bo, ln in plan.export():
        bufs[bb][bo:bo + ln] = bufs[ab][ao:ao + ln]


@pytest.mark.parametrize("k,n1,n2,h", [(4096, 4, 3, 8), (14336, 4, 2, 4), (37, 16, 9, 3),
                                       (96, 8, 8, 2), (32, 4, 1, 4)])
def test_plan_replay_matches_oracle(k, n1, n2, h):
    unit = 2 * h
    contig, sync_l, comp_l = layouts_for_failure(k, n1, n2)
    rng = np.random.default_rng(k)
    src = [rng.standard_normal(len(c) * unit) for c in contig]
    backup = [rng.standard_normal(len(c) * unit) for c in comp_l]
    # degraded replica: contiguous TP-n1 -> sync layout, the last rank died
    dead = (n1 - 1,) if n1 > 1 else ()
    plan = build_reconfig_plan(k, unit, contig, sync_l, torch.float64, dead=dead,
                               backup_cols=comp_l).finalize()
    bufs = [s.copy() for s in src] + [np.zeros(len(c) * unit) for c in sync_l] + \
        [b.copy() for b in backup]
    _replay(plan, bufs)
    want = _oracle_move(src, [len(c) * unit for c in sync_l], contig, sync_l, k, unit,
                        dead=dead, backup=backup, backup_cols=comp_l)
    for got, w in zip(bufs[n1:n1 + n2], want):
        assert np.array_equal(got, w)
    # no unit is read from the dead rank
    tab = plan.export()
    assert not np.isin(tab[:, 0], list(dead)).any()
    # healthy replica: contiguous TP-n1 -> NTP comp layout (no deaths)
    plan = build_reconfig_plan(k, unit, contig, comp_l, torch.float64).finalize()
    bufs = [s.copy() for s in src] + [np.zeros(len(c) * unit) for c in comp_l]
    _replay(plan, bufs)
    want = _oracle_move(src, [len(c) * unit for c in comp_l], contig, comp_l, k, unit)
    for got, w in zip(bufs[n1:], want):
        assert np.array_equal(got, w)


def test_ownership_replay_agrees_with_reference_plans():
    """comp -> sync ownership after the data move equals apply_plan(PRE_SYNC)."""
    for k, n1, n2 in [(4096, 4, 3), (12000, 32, 30), (60, 6, 3)]:
        smap = build_shard_map(k, n1, n2)
        _, sync_l, comp_l = layouts_for_failure(k, n1, n2, smap)
        own_after = ownership_after(smap.comp_rank, sync_l)
        assert np.array_equal(own_after, apply_plan(smap.comp_rank, build_reshard_plan(smap, PRE_SYNC)))
        back = ownership_after(own_after, comp_l)
        assert np.array_equal(back, apply_plan(smap.sync_rank, build_reshard_plan(smap, POST_SYNC)))


def test_contiguous_to_contiguous_runs_follow_interval_overlaps():
    """TP4 -> TP3 contiguous: the merged runs are exactly the interval pieces."""
    from paper_2504_06095_b200.shardmap import interval_overlaps
    from paper_2504_06095_b200.tpnumerics import contiguous_assignment
    k, unit = 14336, 16
    plan = build_reconfig_plan(k, unit, contiguous_assignment(k, 4), contiguous_assignment(k, 3),
                               torch.bfloat16).finalize()
    assert plan.stats["n_runs"] == len(interval_overlaps(k, 4, 3))


def test_dead_rank_requires_backup():
    contig, sync_l, _ = layouts_for_failure(12, 4, 3)
    with pytest.raises(ValueError, match="backup"):
        build_reconfig_plan(12, 4, contig, sync_l, torch.float32, dead=(3,))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_gpu_reconfigure_bit_exact(dtype):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200.reconfig import alloc_layout, reconfigure, reconfigure_state
    k, n1, n2, h = 14336, 4, 3, 64
    unit = 2 * h
    contig, sync_l, comp_l = layouts_for_failure(k, n1, n2)
    g = torch.Generator(device="cuda").manual_seed(3)
    src = [torch.randn(len(c) * unit, generator=g, device="cuda").to(dtype) for c in contig]
    backup = [torch.randn(len(c) * unit, generator=g, device="cuda").to(dtype) for c in comp_l]
    dst = alloc_layout(sync_l, unit, dtype, "cuda")
    plan = build_reconfig_plan(k, unit, contig, sync_l, dtype, dead=(3,),
                               backup_cols=comp_l).finalize()
    reconfigure(src, dst, plan, backup)
    torch.cuda.synchronize()
    to_np = lambda t: t.view(torch.int16 if dtype == torch.bfloat16 else torch.int32).cpu().numpy()  # noqa: E731
    want = _oracle_move([to_np(s) for s in src], [len(c) * unit for c in sync_l], contig, sync_l,
                        k, unit, dead=(3,), backup=[to_np(b) for b in backup], backup_cols=comp_l)
    for got, w in zip(dst, want):
        assert np.array_equal(to_np(got), w)
    # a whole optimizer state set in one call (param bf16 + fp32 master/m/v)
    states = {}
    for name, dt in (("param", torch.bfloat16), ("master", torch.float32),
                     ("exp_avg", torch.float32), ("exp_avg_sq", torch.float32)):
        s = [torch.randn(len(c) * unit, generator=g, device="cuda").to(dt) for c in contig]
        states[name] = (s, alloc_layout(comp_l, unit, dt, "cuda"))
    plans = reconfigure_state(states, k, unit, contig, comp_l)
    assert len(plans) == 2
    torch.cuda.synchronize()
    for name, (s, d) in states.items():
        cat_s = torch.cat(s).view(-1, unit)
        cat_d = torch.cat(d).view(-1, unit)
        order = torch.as_tensor(np.concatenate(comp_l), device="cuda")
        assert torch.equal(cat_d, cat_s[order])
