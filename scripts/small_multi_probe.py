"""Where does a small cross-GPU sync step spend its time?  (torchrun, N=2)

Per-step device time, max over ranks, of NtpSyncGroup steps (CUDA-graph
replays unless noted) for:

  tiny          a 2-unit workload: the handshake + launch floor
  c1_noflush    the C1 workload (h1024/ffn4096 fp32, 33.5 MB per replica)
  c1_wflush     C1 after a 256 MB L2 write-flush (fill_) in the same graph
  c1_rflush     C1 after a 256 MB L2 read-flush (sum) in the same graph
  c1_wflush_sync  write-flush, device sync + barrier, then the step (eager)

    torchrun --nproc-per-node 2 scripts/small_multi_probe.py
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.workloads import C1, ModelShape, pair_layout  # noqa: E402


def dmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = dist.get_world_size()
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    acc = torch.empty(1, dtype=torch.int64, device="cuda")
    fl_w = lambda: flush.fill_(1)  # noqa: E731
    fl_r = lambda: acc.copy_(flush.view(torch.int64).sum())  # noqa: E731
    out = {}
    for name, shape, dt in (("tiny", ModelShape("tiny", 64, 8, 0, 1), torch.float32),
                            ("c1", C1, torch.float32)):
        lay = pair_layout(shape, 4, 3)
        grp = NtpSyncGroup(lay, Placement.default(world, 4, 3), dt, device=local).upload()
        for sl in grp.hosted:
            grp.arena(sl).normal_()
        cases = {"graph": lambda: grp.step_graph(4 / 7, 3 / 7, s),
                 "graph_fused": None,
                 "eager": lambda: grp.step(4 / 7, 3 / 7, s)}
        if name == "c1":
            cases.update({
                "graph_wflush": lambda: grp.step_graph(4 / 7, 3 / 7, s, prologue=fl_w),
                "graph_rflush": lambda: grp.step_graph(4 / 7, 3 / 7, s, prologue=fl_r),
                "wflush_only": fl_w, "rflush_only": fl_r})
        for case, fn in cases.items():
            if case == "graph_fused":
                grp.fused_step = True
                fn = lambda: grp.step_graph(4 / 7, 3 / 7, s)  # noqa: E731
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(50):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            out[f"{name}_{case}_us"] = round(dmax(e0.elapsed_time(e1) / 50) * 1e3, 2)
            grp.fused_step = False
        if name == "c1":  # flush + host sync + barrier, then one eager step, timed alone
            ts = []
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(30):
                fl_w()
                torch.cuda.synchronize()
                dist.barrier()
                e0.record(s)
                grp.step(4 / 7, 3 / 7, s)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(dmax(e0.elapsed_time(e1)))
            ts.sort()
            out["c1_wflush_sync_eager_us_median"] = round(ts[len(ts) // 2] * 1e3, 2)
        assert grp.status() == 0
        dist.barrier()
        grp.close()
    if dist.get_rank() == 0:
        print(json.dumps(out, indent=1), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
