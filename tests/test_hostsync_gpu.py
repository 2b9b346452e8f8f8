"""HostSync: the host-buffer API of the sync (hostsync.py), pipelined per layer
over two copy streams, run several times back to back so that run i+1's
host-to-device copies overlap run i's device-to-host tail.  Each run must see
the previous run's results: with the plain sum (weights 1, 1) three runs give
4 * (a + b) on every unit of both replicas (exact in fp32)."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("back_to_back", [False, True], ids=["ordered", "back_to_back"])
def test_back_to_back_runs_see_previous_results(back_to_back):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200.hostsync import HostSync
    from paper_2504_06095_b200.workloads import ModelShape, build_plan, layer_pieces, pair_layout
    shape = ModelShape("tiny", hidden=64, ffn=600, heads=4, layers=6)
    lay = pair_layout(shape, 4, 3)
    dt = torch.float32
    plan = build_plan(lay, dt)
    hs = HostSync(plan, list(lay.h_elems) + list(lay.r_elems), dt, device=0,
                  piece_plans=layer_pieces(lay, dt, 0), back_to_back=back_to_back)
    rng = np.random.default_rng(3)
    init = [np.round(rng.standard_normal(e) * 64) / 64 for e in list(lay.h_elems) + list(lay.r_elems)]
    host = [torch.from_numpy(a).to(dt).pin_memory() for a in init]
    for _ in range(3):
        hs.run(host, 1.0, 1.0)
    torch.cuda.synchronize()
    # oracle: one sum-sync, then x4 (runs 2 and 3 double the identical copies)
    hb = [a.copy() for a in init[:lay.n1]]
    rb = [a.copy() for a in init[lay.n1:]]
    for k, unit, hc, rc, hbase, rbase in lay.segs:
        comp = np.empty(k, dtype=np.int64)
        sync = np.empty(k, dtype=np.int64)
        for r, c in enumerate(hc):
            comp[c] = r
        for r, c in enumerate(rc):
            sync[c] = r
        hv = [hb[r][hbase[r]:hbase[r] + len(c) * unit].copy() for r, c in enumerate(hc)]
        rv = [rb[r][rbase[r]:rbase[r] + len(c) * unit].copy() for r, c in enumerate(rc)]
        O.nonuniform_sync(comp, sync, hc, rc, hv, rv, unit, op=O.OP_SUM)
        for r, c in enumerate(hc):
            hb[r][hbase[r]:hbase[r] + len(c) * unit] = hv[r]
        for r, c in enumerate(rc):
            rb[r][rbase[r]:rbase[r] + len(c) * unit] = rv[r]
    for got, want in zip(host, hb + rb):
        assert np.array_equal(got.numpy().astype(np.float64), 4.0 * want)


def test_ordered_run_sees_stream_ordered_host_writes():
    """Default ordering: a non_blocking device->host copy the caller queues on
    the current stream between two runs (refilling the pinned inputs) lands
    before the second run's host->device copies read them."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200.hostsync import HostSync
    from paper_2504_06095_b200.workloads import ModelShape, build_plan, layer_pieces, pair_layout
    shape = ModelShape("tiny", hidden=64, ffn=600, heads=4, layers=6)
    lay = pair_layout(shape, 4, 3)
    dt = torch.float32
    elems = list(lay.h_elems) + list(lay.r_elems)
    hs = HostSync(build_plan(lay, dt), elems, dt, device=0, piece_plans=layer_pieces(lay, dt, 0))
    host = [torch.ones(e, dtype=dt).pin_memory() for e in elems]
    hs.run(host, 1.0, 1.0)
    # a slow device producer, then the refill of every host arena with 3.0
    big = torch.randn(4096, 4096, device="cuda")
    for _ in range(20):
        big = big @ big * 1e-3
    fill = [torch.full((e,), 3.0, dtype=dt, device="cuda") + 0 * big[0, 0] for e in elems]
    for h, f in zip(host, fill):
        h.copy_(f, non_blocking=True)
    hs.run(host, 1.0, 1.0)
    torch.cuda.synchronize()
    for h in host:
        assert torch.all(h == 6.0)
