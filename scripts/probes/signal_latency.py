"""Cross-GPU signal round trip (torchrun, N=2): rank 0 posts ready[e] and waits
for rank 1's, rank 1 waits then posts -- a ping-pong of the sync's handshake
kernels (ntp_signal_post / ntp_signal_wait, st.release.sys / ld.acquire.sys
on IPC-mapped signal pages), K round trips recorded into one CUDA graph.
Also the same K handshakes with rank 0 only posting (one-way launch floor)."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def main():
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    lay = pair_layout(ModelShape("tiny", 64, 8, 0, 1), 4, 3)
    grp = NtpSyncGroup(lay, Placement.default(2, 4, 3), torch.float32, device=local).upload()
    K = 200
    out = {}
    for name in ("pingpong", "post_only"):
        base = grp.epoch
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            for i in range(1, K + 1):
                e = base + i
                if name == "post_only":
                    grp.signal("post_ready", e, s)
                elif rank == 0:
                    grp.signal("post_ready", e, s)
                    grp.signal("wait_ready", e, s)
                else:
                    grp.signal("wait_ready", e, s)
                    grp.signal("post_ready", e, s)
        grp.epoch = base + K
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / K * 1e3], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[f"{name}_us_per_iter"] = round(float(t.item()), 3)
    assert grp.status() == 0
    if rank == 0:
        print(json.dumps(out), flush=True)
    grp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
