"""Host logic of the DP > 2 group (dist_dp.NtpDpGroup) on CPU: a real gloo group
(world 4) with a fake device layer.  Across all healthy processes, the fold-in
/ push-back plans must cover every unit of the degraded replica exactly once,
each inside its (piece, replica) sub-range; on every healthy arena the folded
and the scale-only units of each piece must tile the piece exactly once --
which is what makes the plain NCCL SUM of phase B correct and lets piece p's
all-reduce start right after piece p's phase A."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_06095_b200 import dist_dp as DD
from test_dist_host import FakeOps, _free_port

K, UNIT = 3000, 128


def _worker(rank, world, port, m, n1, n2, pieces, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plc = DD.DpPlacement.default(world, m, n1, n2)
    w = np.array([n1] * m + [n2], dtype=np.float64)
    g = DD.NtpDpGroup(K, UNIT, m, plc, torch.float32, 0, w / w.sum(), ops=FakeOps(rank),
                      pieces=pieces)
    order = sorted(g.slot_ptr)
    ex = lambda ps: [p.export() if p is not None else np.zeros((0, 5), dtype=np.int64)  # noqa: E731
                     for p in ps]
    q.put((rank, ex(g.plans), ex(g.scale_plans), order, [b.tolist() for b in g.bounds],
           g.partners, g.replica, g.is_d))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, m, n1, n2, pieces):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, m, n1, n2, pieces, q))
          for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {o[0]: o[1:] for o in out}


@pytest.mark.parametrize("world,m,pieces", [(4, 2, 1), (4, 2, 5), (4, 3, 4), (7, 3, 3)])
def test_gloo_dp_plans_cover_degraded_units_once(world, m, pieces):
    n1, n2 = 2, 1
    per = _run(world, m, n1, n2, pieces)
    d_slot0 = m * n1
    covered_d = np.zeros(K * UNIT, dtype=np.int32)  # the degraded (TP1) arena
    tiles = {}
    for rank, (folds, scales, order, bounds, partners, replica, is_d) in per.items():
        assert len(folds) == pieces and len(scales) == pieces
        if replica is None:
            assert all(len(t) == 0 for t in folds + scales)
            continue
        for pc in range(pieces):
            for ab, ao, bb, bo, ln in folds[pc]:
                a_slot, b_slot = order[ab], order[bb]
                r, i = divmod(a_slot, n1)
                assert r == replica and b_slot == d_slot0
                lo, hi = bounds[i][pc], bounds[i][pc + 1]
                sa, sb = lo + (hi - lo) * r // m, lo + (hi - lo) * (r + 1) // m
                assert sa * UNIT <= ao and ao + ln <= sb * UNIT   # inside its sub-range
                covered_d[bo:bo + ln] += 1
                t = tiles.setdefault(a_slot, {})
                t.setdefault(pc, []).append((ao, ao + ln))
            for ab, ao, bb, bo, ln in scales[pc]:
                assert ab == bb and ao == bo                       # x <- w_r * x in place
                a_slot = order[ab]
                i = a_slot % n1
                lo, hi = bounds[i][pc] * UNIT, bounds[i][pc + 1] * UNIT
                assert lo <= ao and ao + ln <= hi
                tiles.setdefault(a_slot, {}).setdefault(pc, []).append((ao, ao + ln))
    assert (covered_d == 1).all()
    for a_slot, by_piece in tiles.items():      # fold + scale tile each piece once
        i = a_slot % n1
        bounds = per[0][3][i]
        for pc, spans in by_piece.items():
            spans.sort()
            assert spans[0][0] == bounds[pc] * UNIT and spans[-1][1] == bounds[pc + 1] * UNIT
            assert all(x[1] == y[0] for x, y in zip(spans, spans[1:]))
    # every healthy replica takes part in the fold (the work is spread)
    assert {v[5] for v in per.values() if v[5] is not None} == set(range(m))
    d_rank = [r for r, v in per.items() if v[-1]][0]
    assert sorted(per[d_rank][4]) == sorted(r for r, v in per.items() if v[5] is not None)


def test_pieces_validated():
    with pytest.raises(ValueError, match="pieces"):
        DD.NtpDpGroup(K, UNIT, 2, DD.DpPlacement.default(4, 2, 2, 1), torch.float32, 0,
                      [0.4, 0.4, 0.2], ops=FakeOps(0), pieces=0)


def _multi_worker(rank, world, port, m, n1, n2, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plc = DD.DpPlacement.default(world, m, n1, n2)
    w = np.array([n1] * m + [n2], dtype=np.float64)
    g = DD.NtpDpMultiGroup(K, UNIT, m, plc, torch.float32, 0, w / w.sum(), ops=FakeOps(rank))
    q.put((rank, g.units, g.partners, list(g.hosted)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(4, 3), (4, 2), (7, 3)])
def test_gloo_dp_multi_executes_every_unit_once(world, m):
    """One-shot R-way group: every column executed by exactly one process (one
    of its owners), work spread over all replicas, partner sets symmetric."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_multi_worker, args=(r, world, port, m, 2, 1, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {o[0]: o[1:] for o in (q.get(timeout=120) for _ in range(world))}
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(v[0] for v in out.values()) == K
    # water-filled loads: held + (R-2) * executed; the degraded GPU holds the
    # most, so the max load is that GPU's own holdings (nothing executed there)
    R = m + 1
    held = {r: 0 for r in out}
    plc = DD.DpPlacement.default(world, m, 2, 1)
    for r in range(m):
        for i in range(2):
            held[plc.hp[r][i]] += K // 2
    held[plc.dp[0]] += K
    loads = {r: held[r] + (R - 2) * out[r][0] for r in out}
    holders = [r for r in held if held[r]]
    lower = max(max(held.values()), (sum(held.values()) + (R - 2) * K) / len(holders))
    assert max(loads.values()) <= 1.02 * lower + R
    for r, (_u, partners, _h) in out.items():
        for p in partners:
            assert r in out[p][1]


def test_balanced_executors_equal_replicas():
    """One replica per GPU, equal holdings: every GPU executes k / R units."""
    k, R = 1200, 4
    proc = np.tile(np.arange(R)[:, None], (1, k))
    ex = DD.balanced_executors(proc)
    assert sorted(np.bincount(ex).tolist()) == [k // R] * R
    # runs are contiguous per owner
    assert (np.diff(ex) != 0).sum() == R - 1
