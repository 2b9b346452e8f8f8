"""Host logic of the multi-GPU failure reconfiguration (dist_reconfig.py) on
CPU: a real gloo group (world 2 and 4) with a fake device layer.  Every
process's pull table is replayed on numpy arenas; the union must place every
column exactly once in each destination layout, take the dead rank's columns
from the healthy replica and everything else from the replica's own copy --
the ownership algebra of build_shard_map / contiguous_assignment
(shardmap.py:141-182, tpnumerics.py:115-128)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_06095_b200 import dist_reconfig as R
from paper_2504_06095_b200.shardmap import build_shard_map
from paper_2504_06095_b200.tpnumerics import (assignment_from_comp, assignment_from_sync,
                                              contiguous_assignment)
from test_dist_host import FakeOps, _free_port

SEGS = ((96, 32), (12, 64), (96, 32))  # layer MLP columns, heads, next layer


def _worker(rank, world, port, n1, n2, dead, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lay = R.FailureLayout(n1, n2, dead, SEGS)
    proc = R.failure_placement(n1, dead, world)
    g = R.DistReconfig(lay, proc, {"param": torch.bfloat16, "master": torch.float32}, device=0,
                       ops=FakeOps(rank))
    tabs = {str(dt): p.export() for dt, p in g.plans.items()}
    order = sorted(g.buf_index, key=g.buf_index.get)
    q.put((rank, tabs, order, g.hosted, g.units, g.bytes_pulled()))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, n1, n2, dead):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n1, n2, dead, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {o[0]: o[1:] for o in out}


def _expected(lay, arenas):
    """Destination arenas built column by column from the layouts."""
    n1, n2 = lay.n1, lay.n2
    want = {s: np.zeros(e) for s, e in enumerate(lay.slot_elems())}
    base = np.zeros(lay.n_slots(), dtype=np.int64)
    for k, unit in lay.segs:
        smap = build_shard_map(k, n1, n2)
        contig = contiguous_assignment(k, n1)
        comp, sync = assignment_from_comp(smap), assignment_from_sync(smap)

        def where(cols_per_rank, slot0, c):
            for r, cols in enumerate(cols_per_rank):
                hit = np.flatnonzero(np.asarray(cols) == c)
                if len(hit):
                    return slot0 + r, int(base[slot0 + r]) + int(hit[0]) * unit
            raise AssertionError

        for c in range(k):
            hs, ho = where(contig, 0, c)
            ds, do = where(contig, n1, c)
            src_d = (hs, ho) if ds - n1 == lay.dead else (ds, do)
            ts, to = where(comp, 2 * n1, c)
            want[ts][to:to + unit] = arenas[hs][ho:ho + unit]
            ts, to = where(sync, 3 * n1, c)
            want[ts][to:to + unit] = arenas[src_d[0]][src_d[1]:src_d[1] + unit]
        for i in range(n1):
            base[i] += len(contig[i]) * unit
            if i != lay.dead:
                base[n1 + i] += len(contig[i]) * unit
            base[2 * n1 + i] += len(comp[i]) * unit
        for j in range(n2):
            base[3 * n1 + j] += len(sync[j]) * unit
    return want


def _merged(tab):
    """Chunk records (a_buf, a_off, b_buf, b_off, len) merged into maximal runs
    that are contiguous on both sides."""
    runs = []
    for ab, ao, bb, bo, ln in sorted(map(tuple, np.asarray(tab).tolist())):
        if runs and runs[-1][0] == ab and runs[-1][2] == bb and \
                runs[-1][1] + runs[-1][4] == ao and runs[-1][3] + runs[-1][4] == bo:
            runs[-1][4] += ln
        else:
            runs.append([ab, ao, bb, bo, ln])
    return runs


@pytest.mark.parametrize("world,n1,dead", [(2, 4, 3), (2, 4, 0), (4, 2, 1), (4, 4, 1)])
def test_gloo_failure_reconfig_tables(world, n1, dead):
    n2 = n1 - 1
    per_rank = _run(world, n1, n2, dead)
    lay = R.FailureLayout(n1, n2, dead, SEGS)
    rng = np.random.default_rng(world * 10 + n1 + dead)
    elems = lay.slot_elems()
    arenas = [rng.standard_normal(e) for e in elems]
    got = [a.copy() for a in arenas]
    for s in range(2 * n1, lay.n_slots()):
        got[s][:] = np.nan
    covered = [np.zeros(e, dtype=np.int32) for e in elems]
    proc = R.failure_placement(n1, dead, world)
    for rank, (tabs, order, hosted, units, nbytes) in per_rank.items():
        if not any(proc[d] == rank for d in range(2 * n1, lay.n_slots())):
            assert tabs == {} and units == 0       # e.g. the dead GPU's process: no work
            continue
        assert set(tabs) == {str(torch.bfloat16), str(torch.float32)}
        t16, t32 = tabs[str(torch.bfloat16)], tabs[str(torch.float32)]
        # the same units move in every dtype (chunk boundaries may differ: a
        # chunk is a byte budget, NTP_OPT_PLAN_MIN_CHUNKS splits small plans)
        assert _merged(t16) == _merged(t32)
        for ab, ao, bb, bo, ln in t16:
            src, dst = order[ab], order[bb]
            assert proc[dst] == rank                 # pull model: destinations are local
            assert src != n1 + dead                  # never the dead GPU
            assert dst >= 2 * n1                     # sources are never written
            got[dst][bo:bo + ln] = arenas[src][ao:ao + ln]
            covered[dst][bo:bo + ln] += 1
        # bytes accounting: bf16 + fp32 of every pulled element
        assert nbytes["local"] + nbytes["peer"] == int(t16[:, 4].sum()) * 6
    for s in range(2 * n1, lay.n_slots()):
        assert (covered[s] == 1).all()
    want = _expected(lay, arenas)
    for s in range(2 * n1, lay.n_slots()):
        np.testing.assert_array_equal(got[s], want[s])


def test_dead_slot_has_no_arena_and_bad_degree_rejected():
    lay = R.FailureLayout(4, 3, 2, SEGS)
    assert lay.slot_elems()[4 + 2] == 0
    with pytest.raises(ValueError, match="TP4 to TP3, not TP2"):
        R.FailureLayout(4, 2, 2, SEGS).units()


def test_placement_keeps_survivors_on_their_gpus():
    proc = R.failure_placement(4, 1, 8)
    assert proc[:4] == [0, 1, 2, 3] and proc[4:8] == [4, 5, 6, 7]
    assert proc[8:12] == [0, 1, 2, 3]              # H_dst where H_src was
    assert proc[12:] == [4, 6, 7]                  # survivors 0, 2, 3 of D
