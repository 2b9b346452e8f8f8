"""DP > 2 with one degraded replica (BASELINE configs[2] shape: DP=4 x TP2, one
replica degraded to TP1), run under torchrun.  m healthy TP-n1 replicas + one
degraded TP-n2 replica through dist_dp.NtpDpGroup; the gradient is the MLP part
of the GPT-1.3B-shaped model (24 layers x ffn 8192 columns, unit 2h, bf16) as
one unit-major partition.  Device time per step (max over ranks), the
degraded GPU's link bytes, and NCCL's all-reduce of the same bytes across all
m+1 replicas (the uniform-DP comparator).  JSON on rank 0.

    torchrun --nproc-per-node 4 scripts/dp_bench.py [m n1 n2 steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200.dist_dp import DpPlacement, NtpDpGroup  # noqa: E402  (and NtpDpMultiGroup below)


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n1 = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    n2 = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    piece_list = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [1, 4, 8, 16]
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    h, ffn, layers = 2048, 8192, 24
    k, unit = ffn * layers, 2 * h
    batches = [n1] * m + [n2]
    w = np.array(batches, dtype=np.float64) / sum(batches)
    plc = DpPlacement.default(world, m, n1, n2)
    stream = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(rank)

    def timed(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return tmax(e0.elapsed_time(e1) / iters)

    from paper_2504_06095_b200 import _lib
    Lb = _lib.load()
    # sync-kernel settings: (variant, CTA cap) -- a capped kernel leaves SMs to
    # the NCCL all-reduce of the previous piece running beside it
    settings = [(0, 0), (2, 64), (2, 32), (1, 64)]
    by_pieces = {}
    for pieces in piece_list:
        grp = NtpDpGroup(k, unit, m, plc, torch.bfloat16, local, w, pieces=pieces).upload()
        for s in grp.hosted:
            a = grp.arena(s)
            a.copy_(torch.randn(a.numel(), generator=g, device="cuda").to(torch.bfloat16))
        for kern, cap in settings if pieces > 1 else settings[:1]:
            Lb.ntp_set_option(0, kern)
            Lb.ntp_set_option(1, cap)
            by_pieces[f"{pieces}/k{kern}c{cap}"] = timed(lambda: grp.step(stream), steps)
        Lb.ntp_set_option(0, 0)
        Lb.ntp_set_option(1, 0)
        assert grp.status() == 0, "signal timeout"
        grp.close()
    # one R-way peer-memory kernel per process (no NCCL)
    from paper_2504_06095_b200.dist_dp import NtpDpMultiGroup
    grp = NtpDpMultiGroup(k, unit, m, plc, torch.bfloat16, local, w).upload()
    for s in grp.hosted:
        a = grp.arena(s)
        a.copy_(torch.randn(a.numel(), generator=g, device="cuda").to(torch.bfloat16))
    for variant, name in ((1, "multi_ldg"), (2, "multi_bulk")):
        Lb.ntp_multi_set_kernel(variant)
        by_pieces[name] = timed(lambda: grp.step(stream), steps)
    Lb.ntp_multi_set_kernel(0)
    assert grp.status() == 0, "signal timeout"
    grp.close()
    best = min(by_pieces, key=by_pieces.get)
    ms = by_pieces[best]
    eb = 2
    s_d = k * unit * eb  # the degraded replica's whole gradient
    # comparator: uniform DP over the same GPUs, one replica per GPU -- NCCL
    # all-reduce of a whole replica gradient across every rank
    x = torch.randn(k * unit, generator=g, device="cuda").to(torch.bfloat16)
    ms_ar = timed(lambda: dist.all_reduce(x), steps)
    if rank == 0:
        print(json.dumps({
            "workload": f"gpt-1.3b MLP gradients ({layers} x ffn {ffn}, unit 2h, bf16), "
                        f"DP={m + 1}: {m} x TP{n1} + 1 x TP{n2}",
            "n_gpus": world, "placement_healthy": [list(p) for p in plc.hp],
            "placement_degraded": list(plc.dp), "grad_bytes_per_replica": s_d,
            "ms_per_step": round(ms, 3), "pieces": best,
            "ms_by_pieces/kernel/cap": {p: round(v, 3) for p, v in by_pieces.items()},
            # one replica per GPU: every GPU moves 2 (R-1)/R * S per direction
            "per_gpu_bytes_per_direction": int(2 * m / (m + 1) * s_d),
            "per_gpu_GBps_per_direction": round(2 * m / (m + 1) * s_d / (ms * 1e-3) / 1e9, 1),
            "link_frac_of_770": round(2 * m / (m + 1) * s_d / (ms * 1e-3) / 1e9 / 770.0, 3),
            "uniform_dp_nccl_allreduce_ms": round(ms_ar, 3),
            "overhead_vs_uniform_dp": round(ms / ms_ar - 1.0, 4),
            "note": "multi_*: one R-way peer-memory kernel per GPU (NtpDpMultiGroup; "
                    "ldg or TMA-bulk ring); p/kKcC: the NCCL composition (NtpDpGroup) with p "
                    "pipeline pieces and sync kernel K capped at C CTAs"}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
