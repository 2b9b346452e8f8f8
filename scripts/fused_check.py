"""Multi-GPU parity of the fused wgrad GEMM + NTP sync (torchrun, >= 2 ranks).

Every process runs its hosted shards' tcgen05 backward with the fused sync
epilogue: mode "red" red.adds into its own unit-major arena and the partner
replica's (peer HBM); "push" / "push_tma" store into the partner's staging
arena (row stores / TMA tensor stores over NVLink) and each side then adds its
staging locally.  Rank 0 gathers the arenas and compares the dense result with
the fp64 oracle w_h * mlp_backward(X_h) + w_r * mlp_backward(X_r)
(tpnumerics.py:220-235); the two replicas' copies must be bit-identical.

    torchrun --nproc-per-node N scripts/fused_check.py [n1 n2 mode]
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
from paper_2504_06095_b200.linear import MlpShard, finish_push, partner_row_map  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


class _P:
    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


def main():
    n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n2 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    mode = sys.argv[3] if len(sys.argv) > 3 else "red"
    os.environ["NCCL_DEBUG"] = "WARN"
    local = _procgroup.init()
    rank, world = dist.get_rank(), dist.get_world_size()
    h, k, tok_h = 256, 1000, 512
    tok_r = tok_h * n2 // n1
    w_h, w_r = tok_h / (tok_h + tok_r), tok_r / (tok_h + tok_r)
    lay = pair_layout(ModelShape("fused", h, k, 0, 1), n1, n2)
    plc = Placement.default(world, n1, n2)
    grp = NtpSyncGroup(lay, plc, torch.float32, local).upload()
    stg = NtpSyncGroup(lay, plc, torch.float32, local).upload() if mode in ("push", "push_tma") else None
    _, unit, hc, rc, _, _ = lay.segs[0]
    rng = np.random.default_rng(5)  # identical on every rank
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    r64 = lambda x: bf(x).double().numpy()  # noqa: E731
    A, B = r64(rng.standard_normal((h, k)) / np.sqrt(h)), r64(rng.standard_normal((k, h)) / np.sqrt(k))
    Xh, Gh = r64(rng.standard_normal((tok_h, h))), r64(rng.standard_normal((tok_h, h)))
    Xr, Gr = r64(rng.standard_normal((tok_r, h))), r64(rng.standard_normal((tok_r, h)))
    work = []
    for s in grp.hosted:
        healthy = s < n1
        cols = hc[s] if healthy else rc[s - n1]
        X, G = (Xh, Gh) if healthy else (Xr, Gr)
        sh = MlpShard(A, B, cols)
        sh.forward(bf(X).cuda(), torch.empty((X.shape[0], h), device="cuda"))
        slots = [n1 + j for j in range(n2)] if healthy else list(range(n1))
        ptrs = (grp if mode in ("red", "red_tma") else stg).open_slots(slots)
        rb, rr = partner_row_map(cols, rc if healthy else hc, "cuda")
        work.append((sh, bf(X).cuda(), bf(G).cuda(), grp.arena(s).view(len(cols), 2, h),
                     w_h if healthy else w_r, rb, rr, ptrs, s))
    e = 1
    if mode in ("red", "red_tma"):
        for s in grp.hosted:
            grp.arena(s).zero_()
    grp.signal("post_ready", e)
    grp.signal("wait_ready", e)
    for sh, X, G, grads, alpha, rb, rr, ptrs, _s in work:
        sh.backward_synced(X, G, grads, alpha, rb, rr, [_P(p) for p in ptrs], mode=mode)
    grp.signal("post_done", e)
    grp.signal("wait_done", e)
    if stg is not None:
        for sh, X, G, grads, alpha, rb, rr, ptrs, s in work:
            finish_push(grp.arena(s), stg.arena(s))
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
        da1, db1 = O.mlp_backward(Xh, A, B, Gh)
        da2, db2 = O.mlp_backward(Xr, A, B, Gr)
        want_a, want_b = w_h * da1 + w_r * da2, w_h * db1 + w_r * db2
        worst = 0.0
        dense = {}
        for s in range(n1 + n2):
            cols = hc[s] if s < n1 else rc[s - n1]
            u = got[s].reshape(len(cols), 2 * h)
            ga, gb = u[:, :h].T, u[:, h:]
            worst = max(worst, O.rel_err(ga, want_a[:, cols]), O.rel_err(gb, want_b[cols, :]))
            for p, c in enumerate(cols):
                dense.setdefault(int(c), []).append(u[p])
        same = all(np.array_equal(v[0], v[1]) for v in dense.values())
        ok = worst < 2e-2 and same
        print(f"fused_check {mode} world={world} n1={n1} n2={n2} worst_rel_err={worst:.3e} "
              f"replicas_identical={same} {'PASS' if ok else 'FAIL'}", flush=True)
    grp.close()
    if stg is not None:
        stg.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
