"""DP > 2 multi-GPU parity check (torchrun, >= 3 ranks): m healthy TP-n1
replicas + one degraded TP-n2 replica through dist_dp.NtpDpGroup, compared with
the oracle's uniform_sync arithmetic on dense layouts.

    torchrun --nproc-per-node 4 scripts/dp_check.py [m n1 n2 dtype steps pieces algo]

algo "nccl" (default): fold-in / NCCL all-reduce / push-back (NtpDpGroup);
"multi": one R-way peer-memory kernel per process (NtpDpMultiGroup).
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import _procgroup  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2504_06095_b200.dist_dp import DpPlacement, NtpDpGroup, NtpDpMultiGroup  # noqa: E402

DT = {"f32": torch.float32, "bf16": torch.bfloat16}
TOL = {"f32": 1e-6, "bf16": 2e-2}


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n1 = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    n2 = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    dname = sys.argv[4] if len(sys.argv) > 4 else "f32"
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    pieces = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    algo = sys.argv[7] if len(sys.argv) > 7 else "nccl"
    os.environ["NCCL_DEBUG"] = "WARN"
    local = _procgroup.init()
    rank, world = dist.get_rank(), dist.get_world_size()
    k, h = 3000, 64
    unit = 2 * h
    dtype = DT[dname]
    batches = [n1] * m + [n2]  # local batch proportional to TP degree
    w = np.array(batches, dtype=np.float64) / sum(batches)
    plc = DpPlacement.default(world, m, n1, n2)
    if algo == "multi":
        grp = NtpDpMultiGroup(k, unit, m, plc, dtype, local, w).upload()
    else:
        grp = NtpDpGroup(k, unit, m, plc, dtype, local, w, pieces=pieces).upload()
    rng = np.random.default_rng(0)
    dense = [torch.from_numpy(rng.standard_normal((k, unit))).to(dtype).double().numpy()
             for _ in range(m + 1)]

    def cols_of(s):
        return grp.h_cols[s % n1] if s < m * n1 else grp.d_cols[s - m * n1]

    def rep_of(s):
        return s // n1 if s < m * n1 else m

    for s in grp.hosted:
        grp.arena(s).copy_(torch.from_numpy(dense[rep_of(s)][cols_of(s)].ravel()).to(dtype))
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(steps):
        grp.step()
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
        want = [d.ravel().copy() for d in dense]
        for _ in range(steps):
            O.uniform_sync(want, op=O.OP_WEIGHTED, weights=w)
            want = [torch.from_numpy(x).to(dtype).double().numpy() for x in want]
        ref = want[0].reshape(k, unit)
        worst = 0.0
        for s in range(m * n1 + n2):
            dense_got = np.zeros((k, unit))
            dense_got[cols_of(s)] = got[s].reshape(-1, unit)
            worst = max(worst, O.rel_err(dense_got[cols_of(s)], ref[cols_of(s)]))
        ok = worst <= TOL[dname]
        print(f"dp_check world={world} m={m} n1={n1} n2={n2} {dname} steps={steps} "
              f"worst_rel_err={worst:.3e} {'PASS' if ok else 'FAIL'}", flush=True)
    grp.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
