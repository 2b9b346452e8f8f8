"""Host logic of the multi-GPU sync (paper_2504_06095_b200/dist.py) on CPU:
placement, per-process plans, IPC-handle exchange over a real gloo process
group (world size 2), and signal wiring.  Device calls are replaced by a fake;
the per-process chunk tables are replayed on numpy arenas and must reproduce
the oracle's nonuniform sync of the whole layout."""

import os
import pickle
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2504_06095_b200 import dist as D
from paper_2504_06095_b200.workloads import ModelShape, pair_layout

SHAPE = ModelShape("tiny", hidden=16, ffn=96, heads=4, layers=3)


class FakeOps:
    """Pointers are (rank, n) pairs encoded as ints; handles are pickles."""

    def __init__(self, rank):
        self.rank, self.n = rank, 0

    def alloc(self, nbytes):
        self.n += 1
        return (self.rank << 32) | self.n

    def handle(self, ptr):
        return pickle.dumps(ptr).ljust(64, b"\0")

    def open(self, handle):
        return pickle.loads(handle.rstrip(b"\0") if handle[-1:] == b"\0" else handle)

    def close(self, ptr):
        pass

    def free(self, ptr):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n1, n2, q, pieces=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lay = pair_layout(SHAPE, n1, n2)
    plc = D.Placement.default(world, n1, n2)
    g = D.NtpSyncGroup(lay, plc, torch.float32, device=0, ops=FakeOps(rank), pieces=pieces)
    if pieces:
        # the piece plans together must do exactly the whole plan's work
        parts = [p.export() for p in g.piece_plans if p is not None]
        tab = np.concatenate(parts) if parts else np.zeros((0, 5), dtype=np.int64)
        whole = g.plan.export() if g.plan is not None else np.zeros((0, 5), dtype=np.int64)
        assert int(tab[:, 4].sum()) == int(whole[:, 4].sum())
        rng = [g.piece_ranges(i) for i in range(len(pieces))]
        for a, b in zip(rng, rng[1:]):  # pieces tile every hosted arena in order
            for s in g.hosted:
                assert a[s][1] == b[s][0]
        for s in g.hosted:
            assert rng[0][s][0] == 0 and rng[-1][s][1] == g.slot_elems[s]
    else:
        tab = g.plan.export() if g.plan is not None else np.zeros((0, 5), dtype=np.int64)
    slots = sorted(g.slot_ptr)
    q.put((rank, tab, slots, g.wait_ready, g.post_done, g.post_ready, g.wait_done,
           g.partners, g.sig))
    dist.barrier()
    dist.destroy_process_group()


def _run_world(world, n1, n2, pieces=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n1, n2, q, pieces))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {o[0]: o[1:] for o in out}


def _replay(lay, per_rank, w=(4 / 7, 3 / 7), seed=0):
    rng = np.random.default_rng(seed)
    arenas = [rng.standard_normal(e) for e in list(lay.h_elems) + list(lay.r_elems)]
    want_h = [a.copy() for a in arenas[:lay.n1]]
    want_r = [a.copy() for a in arenas[lay.n1:]]
    covered = [np.zeros(len(a), dtype=np.int32) for a in arenas]
    for rank, (tab, slots, *_rest) in per_rank.items():
        for ab, ao, bb, bo, ln in tab:
            A, B = arenas[slots[ab]], arenas[slots[bb]]
            v = w[0] * A[ao:ao + ln] + w[1] * B[bo:bo + ln]
            A[ao:ao + ln] = v
            B[bo:bo + ln] = v
            covered[slots[ab]][ao:ao + ln] += 1
            covered[slots[bb]][bo:bo + ln] += 1
    for c in covered:
        assert (c == 1).all()
    # oracle, segment by segment
    for k, unit, hc, rc, hb, rb in lay.segs:
        comp = np.empty(k, dtype=np.int64)
        sync = np.empty(k, dtype=np.int64)
        for r, c in enumerate(hc):
            comp[c] = r
        for r, c in enumerate(rc):
            sync[c] = r
        hv = [want_h[r][hb[r]:hb[r] + len(c) * unit].copy() for r, c in enumerate(hc)]
        rv = [want_r[r][rb[r]:rb[r] + len(c) * unit].copy() for r, c in enumerate(rc)]
        O.nonuniform_sync(comp, sync, hc, rc, hv, rv, unit, op=O.OP_WEIGHTED, weights=w)
        for r, c in enumerate(hc):
            want_h[r][hb[r]:hb[r] + len(c) * unit] = hv[r]
        for r, c in enumerate(rc):
            want_r[r][rb[r]:rb[r] + len(c) * unit] = rv[r]
    for got, want in zip(arenas, want_h + want_r):
        np.testing.assert_allclose(got, want, rtol=1e-14, atol=1e-14)


def _check_wiring(per_rank):
    """Partner sets are symmetric; every posted word is a word its owner waits on."""
    sig_base = {rank: v[-1] for rank, v in per_rank.items()}
    for rank, (_t, _s, wr, pd, pr, wd, partners, sig) in per_rank.items():
        for p in partners:
            assert rank in per_rank[p][6]
        # my posts land in the partner's page at slot = my rank
        assert sorted(pr) == sorted(sig_base[p] + 8 * (D.READY * D.SIG_WORDS + rank) for p in partners)
        assert sorted(pd) == sorted(sig_base[p] + 8 * (D.DONE * D.SIG_WORDS + rank) for p in partners)
        assert sorted(wr) == sorted(sig + 8 * (D.READY * D.SIG_WORDS + p) for p in partners)
        assert sorted(wd) == sorted(sig + 8 * (D.DONE * D.SIG_WORDS + p) for p in partners)


@pytest.mark.parametrize("n1,n2", [(4, 3), (2, 1)])
def test_gloo_world2_plans_and_wiring(n1, n2):
    per_rank = _run_world(2, n1, n2)
    lay = pair_layout(SHAPE, n1, n2)
    _replay(lay, per_rank)
    _check_wiring(per_rank)
    # world 2, split policy: both GPUs push about half of the shared units
    e0 = per_rank[0][0][:, 4].sum()
    e1 = per_rank[1][0][:, 4].sum()
    assert abs(int(e0) - int(e1)) <= 0.1 * (e0 + e1)


def test_reduced_policy_pushes_from_reduced_side():
    lay = pair_layout(SHAPE, 4, 3)
    plc = D.Placement.default(2, 4, 3)
    u0, _ = D.process_plan_units(lay, plc, 0, policy="reduced")
    u1, _ = D.process_plan_units(lay, plc, 1, policy="reduced")
    assert u0 == [] and len(u1) > 0
    with pytest.raises(ValueError):
        D.unit_executors(lay, plc, policy="other")


def test_placements():
    assert D.Placement.default(8, 4, 3) == D.Placement(4, 3, (0, 1, 2, 3), (4, 5, 6))
    assert D.Placement.default(1, 4, 3) == D.Placement(4, 3, (0,) * 4, (0,) * 3)
    assert D.Placement.default(2, 4, 3) == D.Placement(4, 3, (0,) * 4, (1,) * 3)
    p = D.Placement.default(4, 2, 1)
    assert p.h_proc == (0, 1) and p.r_proc == (2,)
    p = D.Placement.default(4, 4, 3)
    assert set(p.h_proc) | set(p.r_proc) == {0, 1, 2, 3}


@pytest.mark.parametrize("world,n1,n2", [(8, 4, 3), (4, 2, 1), (3, 2, 1), (8, 4, 2)])
def test_single_process_emulation_of_larger_worlds(world, n1, n2):
    """Per-process unit selection for worlds we cannot spawn cheaply: every
    unit is computed by exactly one process, and the union equals the oracle."""
    lay = pair_layout(SHAPE, n1, n2)
    plc = D.Placement.default(world, n1, n2)
    per_rank = {}
    for rank in range(world):
        units, touched = D.process_plan_units(lay, plc, rank)
        rows = []
        for unit, hs, ho, rs, ro in units:
            rows += [(h, a, r, b, unit) for h, a, r, b in zip(hs, ho, rs, ro)]
        tab = np.array(rows, dtype=np.int64).reshape(-1, 5)
        per_rank[rank] = (tab, list(range(n1 + n2)))
    _replay(lay, per_rank)


def test_gloo_world8_tp4_tp3_plans_and_wiring():
    """The 8-GPU bench placement: TP4 + TP3 on 7 ranks, rank 7 idle ("failed")."""
    per_rank = _run_world(8, 4, 3)
    lay = pair_layout(SHAPE, 4, 3)
    _replay(lay, per_rank)
    _check_wiring(per_rank)
    assert len(per_rank[7][0]) == 0 and per_rank[7][6] == []  # idle GPU: no work, no partners


def test_busiest_bytes_accounting():
    from paper_2504_06095_b200.dist_bench import busiest_bytes_for
    from paper_2504_06095_b200.workloads import GPT_1_3B
    lay = pair_layout(GPT_1_3B, 4, 3)
    # 8 GPUs: the busiest reduced GPU owns sync shard 0 (2731 MLP cols + 6 heads per layer)
    b8 = busiest_bytes_for(lay, D.Placement.default(8, 4, 3), 2)
    assert b8 == max(lay.r_elems) * 2 == 838926336
    # 2 GPUs: every unit crosses the one link
    assert busiest_bytes_for(lay, D.Placement.default(2, 4, 3), 2) == lay.elems * 2


def test_gloo_world2_per_layer_pieces():
    """Pipelined pieces (one per layer): their plans replay to the oracle and
    their arena ranges tile every hosted arena."""
    nseg = len(SHAPE.segments())
    pieces = [list(range(i * nseg, (i + 1) * nseg)) for i in range(SHAPE.layers)]
    per_rank = _run_world(2, 4, 3, pieces)
    _replay(pair_layout(SHAPE, 4, 3), per_rank)
    lay = pair_layout(SHAPE, 4, 3)
    with pytest.raises(ValueError, match="contiguous range"):
        D.NtpSyncGroup(lay, D.Placement.default(1, 4, 3), torch.float32, 0, ops=FakeOps(0),
                       pieces=[[0, 2]])


@pytest.mark.parametrize("policy", ["healthy", "0.25", 0.75])
def test_executor_policies_cover_every_unit_once(policy):
    """Any executor share: every unit computed by exactly one process, and the
    union replays to the oracle; "healthy" leaves the degraded GPU idle."""
    lay = pair_layout(SHAPE, 4, 3)
    plc = D.Placement.default(2, 4, 3)
    per_rank = {}
    for rank in range(2):
        units, _ = D.process_plan_units(lay, plc, rank, policy=policy)
        rows = []
        for unit, hs, ho, rs, ro in units:
            rows += [(h, a, r, b, unit) for h, a, r, b in zip(hs, ho, rs, ro)]
        per_rank[rank] = (np.array(rows, dtype=np.int64).reshape(-1, 5), list(range(7)))
    _replay(lay, per_rank)
    if policy == "healthy":
        assert len(per_rank[1][0]) == 0  # GPU 1 hosts the reduced replica
    with pytest.raises(ValueError, match="share must be in"):
        D.reduced_share(1.5)
    with pytest.raises(ValueError, match="unknown executor policy"):
        D.reduced_share("nobody")


def test_gloo_world8_pieces_idle_gpu():
    """The 8-GPU bench with per-layer pieces: GPU 7 (the "failed" one) hosts no
    arena and gets no piece plans; the rest replay to the oracle."""
    nseg = len(SHAPE.segments())
    pieces = [list(range(i * nseg, (i + 1) * nseg)) for i in range(SHAPE.layers)]
    per_rank = _run_world(8, 4, 3, pieces)
    _replay(pair_layout(SHAPE, 4, 3), per_rank)
    assert len(per_rank[7][0]) == 0 and per_rank[7][6] == []
