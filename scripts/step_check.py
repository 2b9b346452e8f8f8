"""OverlappedBackward (paper_2504_06095_b200.step) on N GPUs under torchrun:
the overlapped step (GEMMs on the main stream, each layer's sync on a side
stream, healthy-executor policy, capped kernels) must give the same bits as
the plain order -- all GEMMs, then every layer's sync (split policy).

    torchrun --nproc-per-node N scripts/step_check.py [n1 n2 layers]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.linear import MlpShard  # noqa: E402
from paper_2504_06095_b200.step import OverlappedBackward  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def main():
    n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n2 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    h, k, tok = 256, 1200, 512
    lay = pair_layout(ModelShape("stepcheck", h, k, 0, 1), n1, n2)
    plc = Placement.default(world, n1, n2)
    tok_r = tok * n2 // n1
    w_h, w_r = tok / (tok + tok_r), tok_r / (tok + tok_r)
    _k, _u, hc, rc, _hb, _rb = lay.segs[0]
    rng = np.random.default_rng(0)   # same weights everywhere
    g = torch.Generator(device="cuda").manual_seed(1)
    layers, inputs = [], []
    for li in range(L):
        A = rng.standard_normal((h, k)) / np.sqrt(h)
        B = rng.standard_normal((k, h)) / np.sqrt(k)
        grp = NtpSyncGroup(lay, plc, torch.float32, local).upload()
        shards, ins = [], []
        for s in grp.hosted:
            healthy = s < n1
            cols = hc[s] if healthy else rc[s - n1]
            sh = MlpShard(A, B, cols)
            T = tok if healthy else tok_r
            X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
            G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
            sh.forward(X, torch.empty((T, h), dtype=torch.float32, device="cuda"))
            shards.append((sh, grp.arena(s).view(len(cols), 2, h)))
            ins.append((X, G))
        layers.append((grp, shards))
        inputs.append(ins)
    # reference order: all GEMMs, then every layer's sync (split policy)
    for li in reversed(range(L)):
        for (sh, grads), (X, G) in zip(layers[li][1], inputs[li]):
            sh.backward(X, G, grads)
    for li in reversed(range(L)):
        layers[li][0].step(w_h, w_r)
    torch.cuda.synchronize()
    want = [[grads.clone() for _sh, grads in shards] for _grp, shards in layers]
    # the product path, twice (the second run reuses streams, signals, plans)
    ob = OverlappedBackward(layers, w_h, w_r)
    ok = True
    for _ in range(2):
        for _grp, shards in layers:
            for _sh, grads in shards:
                grads.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        ob.run(inputs)
        torch.cuda.synchronize()
        dist.barrier()
        for (grp, shards), w in zip(layers, want):
            assert grp.status() == 0, "signal timeout"
            for (_sh, grads), ref in zip(shards, w):
                ok &= bool(torch.equal(grads, ref))
    t = torch.tensor([int(ok)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(("PASS" if t.item() else "FAIL") + f" world={world} n1={n1} n2={n2} layers={L}",
              flush=True)
    for grp, _ in layers:
        grp.close()
    dist.destroy_process_group()
    sys.exit(0 if t.item() else 1)


if __name__ == "__main__":
    main()
