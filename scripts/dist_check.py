"""Multi-GPU parity check (run under torchrun): every rank syncs its hosted
arenas through NtpSyncGroup (IPC peer memory + device signals); rank 0 gathers
all arenas and compares them with the oracle's fp64 nonuniform sync.

    torchrun --nproc-per-node N scripts/dist_check.py [n1 n2 dtype steps [launch [policy]]]

launch: "fused" (default here, one ntp_grad_sync_step per step), "three" (post
ready / signalled sync / wait done; NtpSyncGroup's default), "alternate", or
"nccl" (n1 == n2: the aligned NCCL all-reduce fall-through), "graph" / "graph_fused"
(CUDA-graph steps interleaved with eager ones) or "graph_multi" (every step in
one graph); policy: the executor policy
("split" default, "healthy": the reduced side computes nothing and only
hand-shakes)
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import _procgroup  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402

DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}
TOL = {"f32": 1e-6, "bf16": 2e-2, "f64": 0.0}


def main():
    n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    n2 = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dname = sys.argv[3] if len(sys.argv) > 3 else "f32"
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    launch = sys.argv[5] if len(sys.argv) > 5 else "fused"
    policy = sys.argv[6] if len(sys.argv) > 6 else "split"
    local = _procgroup.init()
    rank, world = dist.get_rank(), dist.get_world_size()
    shape = ModelShape("check", hidden=256, ffn=1000, heads=8, layers=3)
    lay = pair_layout(shape, n1, n2)
    plc = Placement.default(world, n1, n2)
    dtype = DT[dname]
    grp = NtpSyncGroup(lay, plc, dtype, device=local, policy=policy,
                       aligned="nccl" if launch.startswith("nccl") else "peer",
                       prescaled=launch == "nccl_pre").upload()
    if launch.startswith("nccl"):
        assert grp.aligned == ("nccl" if n1 == n2 else "peer")
    rng = np.random.default_rng(0)
    init = [rng.standard_normal(e) for e in list(lay.h_elems) + list(lay.r_elems)]
    init = [torch.from_numpy(a).to(dtype).double().numpy() for a in init]  # representable
    for s in grp.hosted:
        grp.arena(s).copy_(torch.from_numpy(init[s]).to(dtype))
    torch.cuda.synchronize()
    dist.barrier()
    w = (4 / 7, 3 / 7)
    if launch == "nccl_pre":  # the producer folded the batch weight in (one step)
        assert steps == 1
        for sl in grp.hosted:
            a = grp.arena(sl)
            a.copy_((a.double() * (w[0] if sl < n1 else w[1])).to(dtype))
        torch.cuda.synchronize()
    if launch == "graph_multi":  # all steps recorded into one CUDA graph
        grp.step_graph(*w, steps=steps)
    for i in range(steps if launch != "graph_multi" else 0):
        grp.fused_step = launch in ("fused", "graph_fused") or (launch == "alternate" and i % 2 == 0)
        grp.two_launch = launch == "graph_two"
        if launch.startswith("graph") and i % 2 == 0:
            grp.step_graph(*w)  # graph replays interleaved with eager steps
        else:
            grp.step(*w)
    torch.cuda.synchronize()
    dist.barrier()
    assert grp.status() == 0, "signal timeout"
    mine = {s: grp.arena(s).double().cpu().numpy() for s in grp.hosted}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    ok = True
    if rank == 0:
        got = {}
        for d in allv:
            got.update(d)
        want = [a.copy() for a in init]
        for _ in range(steps):
            for k, unit, hc, rc, hb, rb in lay.segs:
                comp = np.empty(k, dtype=np.int64)
                sync = np.empty(k, dtype=np.int64)
                for r, c in enumerate(hc):
                    comp[c] = r
                for r, c in enumerate(rc):
                    sync[c] = r
                hv = [want[r][hb[r]:hb[r] + len(c) * unit].copy() for r, c in enumerate(hc)]
                rv = [want[n1 + r][rb[r]:rb[r] + len(c) * unit].copy() for r, c in enumerate(rc)]
                O.nonuniform_sync(comp, sync, hc, rc, hv, rv, unit, op=O.OP_WEIGHTED, weights=w)
                for r, c in enumerate(hc):
                    want[r][hb[r]:hb[r] + len(c) * unit] = hv[r]
                for r, c in enumerate(rc):
                    want[n1 + r][rb[r]:rb[r] + len(c) * unit] = rv[r]
            # the device result of each step is rounded to dtype before the next
            want = [torch.from_numpy(a).to(dtype).double().numpy() for a in want]
        worst = 0.0
        for s in range(n1 + n2):
            err = O.rel_err(got[s], want[s])
            worst = max(worst, err)
        ok = worst <= max(TOL[dname], 0.0) if TOL[dname] else all(
            np.array_equal(got[s], want[s]) for s in range(n1 + n2))
        print(f"dist_check world={world} n1={n1} n2={n2} {dname} steps={steps} {launch} {policy} "
              f"worst_rel_err={worst:.3e} {'PASS' if ok else 'FAIL'}", flush=True)
    grp.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
