"""OverlappedBackward (paper_2504_06095_b200.step) on N GPUs under torchrun
(N = 1 too: every logical rank on one GPU): the overlapped step (GEMMs on the
main stream, each layer's sync on a side stream, healthy-executor policy,
capped kernels) must give the same bits as the plain order -- all GEMMs, then
every layer's sync (split policy) -- and match the fp64 oracle: per layer the
dense w_h * mlp_backward(X_h) + w_r * mlp_backward(X_r) (tpnumerics.py:220-235
summed as nonuniform_grad_sync does, 289-356) on the same bf16-rounded
weights and activations, <= 2e-2, in both replicas' layouts.

    torchrun --nproc-per-node N scripts/step_check.py [n1 n2 layers]
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
from paper_2504_06095_b200.linear import MlpShard  # noqa: E402
from paper_2504_06095_b200.step import OverlappedBackward  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def main():
    n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n2 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    os.environ["NCCL_DEBUG"] = "WARN"
    local = _procgroup.init()
    rank, world = dist.get_rank(), dist.get_world_size()
    h, k, tok = 256, 1200, 512
    lay = pair_layout(ModelShape("stepcheck", h, k, 0, 1), n1, n2)
    plc = Placement.default(world, n1, n2)
    tok_r = tok * n2 // n1
    w_h, w_r = tok / (tok + tok_r), tok_r / (tok + tok_r)
    _k, _u, hc, rc, _hb, _rb = lay.segs[0]
    rng = np.random.default_rng(0)   # same weights and activations on every rank
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    layers, inputs, dense = [], [], []
    for li in range(L):
        A = bf(rng.standard_normal((h, k)) / np.sqrt(h)).double().numpy()
        B = bf(rng.standard_normal((k, h)) / np.sqrt(k)).double().numpy()
        XG = {side: [bf(rng.standard_normal((T, h))) for _ in range(2)]
              for side, T in (("h", tok), ("r", tok_r))}
        dense.append((A, B, {sd: [t.double().numpy() for t in v] for sd, v in XG.items()}))
        grp = NtpSyncGroup(lay, plc, torch.float32, local).upload()
        shards, ins = [], []
        for s in grp.hosted:
            healthy = s < n1
            cols = hc[s] if healthy else rc[s - n1]
            sh = MlpShard(A, B, cols)
            X, G = (t.cuda() for t in XG["h" if healthy else "r"])
            sh.activations(X)
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
    # fp64 oracle: rank 0 gathers every hosted arena and checks each layer
    mine = [{s: grads.double().cpu().numpy().reshape(grads.shape[0], -1)
             for s, (_sh, grads) in zip(grp.hosted, shards)} for grp, shards in layers]
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    worst = 0.0
    if rank == 0:
        for li, (A, B, XG) in enumerate(dense):
            got = {}
            for d in allv:
                got.update(d[li])
            want_a, want_b = (w_h * a + w_r * b for a, b in
                              zip(O.mlp_backward(*XG["h"][:1], A, B, XG["h"][1]),
                                  O.mlp_backward(*XG["r"][:1], A, B, XG["r"][1])))
            for side, cols in (("h", hc), ("r", rc)):
                base = 0 if side == "h" else n1
                da, db = O.dense_from_units([got[base + i] for i in range(len(cols))], cols, h, k)
                worst = max(worst, O.rel_err(da, want_a), O.rel_err(db, want_b))
        ok &= worst <= 2e-2
        print(f"oracle worst rel err {worst:.3e}", flush=True)
    t = torch.tensor([int(ok)], device="cpu" if _procgroup.shared() else "cuda")
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
