"""Per-step device times of the cross-GPU sync step, one-launch vs three-launch
(NtpSyncGroup.fused_step), to characterise the one-launch outliers: is a slow
measurement one long step or uniformly slower steps?  torchrun, 2+ GPUs.

    torchrun --nproc-per-node 2 scripts/step_outliers.py [MB] [steps] [repeats]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    repeats = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    _lib.load()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    k = max(8, mb * 2**20 // (2 * 4096 * 2))
    lay = pair_layout(ModelShape(f"o{mb}", 4096, k, 0, 1), 4, 3)
    grp = NtpSyncGroup(lay, Placement.default(world, 4, 3), torch.bfloat16, device=local).upload()
    for s in grp.hosted:
        a = grp.arena(s)
        a.copy_(torch.randn(a.numel(), device="cuda").to(torch.bfloat16))
    out = {"mb": mb, "steps": steps, "runs": []}
    for rep in range(repeats):
        for fused in (True, False):
            grp.fused_step = fused
            for _ in range(3):
                grp.step(4 / 7, 3 / 7)
            torch.cuda.synchronize()
            dist.barrier()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            ev[0].record()
            for i in range(steps):
                grp.step(4 / 7, 3 / 7)
                ev[i + 1].record()
            torch.cuda.synchronize()
            us = np.array([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(steps)])
            t = torch.tensor(us, device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            us = t.cpu().numpy()
            if rank == 0:
                out["runs"].append({"rep": rep, "fused": fused, "mean_us": round(float(us.mean()), 2),
                                    "median_us": round(float(np.median(us)), 2),
                                    "p99_us": round(float(np.percentile(us, 99)), 2),
                                    "max_us": round(float(us.max()), 2),
                                    "n_over_2x_median": int((us > 2 * np.median(us)).sum())})
    assert grp.status() == 0
    if rank == 0:
        print(json.dumps(out, indent=1))
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
