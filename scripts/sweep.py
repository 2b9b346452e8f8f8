"""BASELINE configs[4]: grad-sync message-size sweep (1 MB .. 1 GB per replica)
and TP4 -> TP3 / TP4 -> TP2 reconfiguration of an 8B-shaped parameter set.

With one GPU every logical rank is a buffer on cuda:0 (HBM roofline); under
torchrun with 2+ ranks the sync sweep runs across the GPUs over NVLink
(dist.NtpSyncGroup, the bench's N>1 path).  Prints one JSON document.

    python scripts/sweep.py [--reconfig-layers L]
    torchrun --nproc-per-node N scripts/sweep.py
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.plans import OPS, tensor_ptrs  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, build_plan, pair_layout  # noqa: E402

HBM = 6541.8
NVL = 770.0


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def sync_sweep_local():
    """h=4096 bf16 MLP units (16 KiB), k chosen so S*b spans 1 MB .. 1 GB."""
    rows = []
    for mb in (1, 4, 16, 64, 256, 1024):
        k = max(8, mb * 2**20 // (2 * 4096 * 2))
        shape = ModelShape(f"sweep{mb}", 4096, k, 0, 1)
        lay = pair_layout(shape, 4, 3)
        plan = build_plan(lay, torch.bfloat16).upload(0)
        arenas = [torch.randn(e, device="cuda").to(torch.bfloat16) for e in lay.h_elems + lay.r_elems]
        ptrs = tensor_ptrs(arenas)
        # small messages fit in L2: flush it between launches by timing a chain
        # long enough that the data set is re-streamed; report both honestly
        iters = max(5, min(2000, int(2e9 / (lay.elems * 2))))
        b = 4 * lay.elems * 2
        row = {"grad_bytes_per_replica": lay.elems * 2, "k": k,
               "note": "L2-resident" if b < 100e6 else "HBM-streamed"}
        L = _lib.load()
        for name, v in (("auto", 0), ("ldg", 1), ("bulk", 2)):
            if v:
                _lib.check(L.ntp_set_option(0, v))
            ms = timed(lambda: plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7), iters)
            row[name] = {"us": round(ms * 1e3, 2), "hbm_gbs": round(b / ms / 1e6, 1),
                         "frac_hbm": round(b / ms / 1e6 / HBM, 3)}
        _lib.check(L.ntp_set_option(0, 0))
        rows.append(row)
        del arenas
    return rows


def reconfig(layers):
    """8B-shaped (h4096, ffn14336, 32 heads) parameter set: bf16 params + fp32
    master/exp_avg/exp_avg_sq, contiguous TP4 -> TP3 sync layout (degraded
    replica, rank 3 dead -> sourced from the healthy replica's comp-layout copy)
    and -> TP2, on one GPU (HBM roofline: 2 x bytes moved)."""
    from paper_2504_06095_b200.reconfig import build_reconfig_plan, layouts_for_failure
    from paper_2504_06095_b200.tpnumerics import contiguous_assignment
    h, ffn, heads = 4096, 14336, 32
    out = []
    for n2 in (3, 2):
        res = {"to": f"TP{n2}", "layers": layers}
        for dtype, name in ((torch.bfloat16, "param_bf16"), (torch.float32, "fp32_state_x3")):
            reps = 1 if dtype == torch.bfloat16 else 3
            total_ms = 0.0
            moved = 0
            for k, unit in ((ffn, 2 * h), (heads, 4 * h * (h // heads))):
                contig, sync_l, comp_l = layouts_for_failure(k, 4, n2)
                dst_cols = sync_l if n2 == 3 else contiguous_assignment(k, n2)
                plan = build_reconfig_plan(k, unit, contig, dst_cols, dtype, dead=(3,),
                                           backup_cols=comp_l).finalize().upload(0)
                # one layer's segment (> L2); the layer stack repeats it `layers` times
                src = [torch.empty(len(c) * unit, dtype=dtype, device="cuda") for c in contig]
                dst = [torch.empty(len(c) * unit, dtype=dtype, device="cuda") for c in dst_cols]
                bk = [torch.empty(len(c) * unit, dtype=dtype, device="cuda") for c in comp_l]
                ptrs = tensor_ptrs(src + dst + bk)
                ms = timed(lambda: plan.reshard(ptrs), 20)
                total_ms += ms * layers * reps
                moved += k * unit * dtype.itemsize * layers * reps
                del src, dst, bk
            res[name] = {"ms": round(total_ms, 3), "bytes": moved,
                         "hbm_gbs": round(2 * moved / total_ms / 1e6, 1),
                         "frac_hbm": round(2 * moved / total_ms / 1e6 / HBM, 3)}
        out.append(res)
    return out


def sync_sweep_dist():
    """The same message sizes across processes (torchrun, one per GPU): the 7
    logical ranks placed by Placement.default, NVLink peer-memory sync
    (dist.NtpSyncGroup, the bench's N>1 path), device-timed, max over ranks.
    At N=2 NCCL's all-reduce of one replica's bytes between the two GPUs (what a
    uniform DP=2 sync moves) is timed beside it."""
    import torch.distributed as dist
    from paper_2504_06095_b200.dist import NtpSyncGroup, Placement
    from paper_2504_06095_b200.dist_bench import busiest_bytes_for
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))

    def dmax(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def dtimed(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return dmax(e0.elapsed_time(e1) / iters)

    rows = []
    for mb in (1, 4, 16, 64, 256, 1024):
        k = max(8, mb * 2**20 // (2 * 4096 * 2))
        lay = pair_layout(ModelShape(f"sweep{mb}", 4096, k, 0, 1), 4, 3)
        plc = Placement.default(world, 4, 3)
        grp = NtpSyncGroup(lay, plc, torch.bfloat16, device=local).upload()
        grp.fused_step = os.environ.get("NTP_FUSED_STEP", "0") != "0"  # A/B: 1 vs 3 launches
        for s in grp.hosted:
            a = grp.arena(s)
            a.copy_(torch.randn(a.numel(), device="cuda").to(torch.bfloat16))
        iters = max(5, min(500, int(2e9 / (lay.elems * 2))))
        ms = dtimed(lambda: grp.step(4 / 7, 3 / 7), iters)
        # the same steps as CUDA-graph launches: 3-launch and 1-launch variants
        grp.fused_step = False
        ms_g3 = dtimed(lambda: grp.step_graph(4 / 7, 3 / 7), iters)
        grp.two_launch = True
        ms_g2 = dtimed(lambda: grp.step_graph(4 / 7, 3 / 7), iters)
        grp.two_launch = False
        grp.fused_step = True
        ms_g1 = dtimed(lambda: grp.step_graph(4 / 7, 3 / 7), iters)
        grp.fused_step = os.environ.get("NTP_FUSED_STEP", "0") != "0"
        if grp.status() != 0:
            raise RuntimeError(f"rank {rank}: signal timeout")
        B = busiest_bytes_for(lay, plc, 2)
        best = min(ms_g3, ms_g2, ms_g1)
        row = {"grad_bytes_per_replica": lay.elems * 2, "k": k, "us": round(ms * 1e3, 2),
               "busiest_gpu_bytes_per_direction": B,
               "nvlink_gbs": round(B / ms / 1e6, 1), "frac_nvlink": round(B / ms / 1e6 / NVL, 3),
               "graph3_us": round(ms_g3 * 1e3, 2), "graph2_us": round(ms_g2 * 1e3, 2),
               "graph1_us": round(ms_g1 * 1e3, 2),
               "graph_frac_nvlink": round(B / best / 1e6 / NVL, 3)}
        if world == 2:
            t = torch.randn(lay.elems, device="cuda").to(torch.bfloat16)
            ms_n = dtimed(lambda: dist.all_reduce(t), iters)
            row["nccl_allreduce_us"] = round(ms_n * 1e3, 2)
            del t
        rows.append(row)
        dist.barrier()
        grp.close()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reconfig-layers", type=int, default=32)
    ap.add_argument("--sync-only", action="store_true")
    args = ap.parse_args()
    L = _lib.load()
    if os.environ.get("NTP_MIN_CHUNKS"):  # experiments: NTP_OPT_PLAN_MIN_CHUNKS
        _lib.check(L.ntp_set_option(2, int(os.environ["NTP_MIN_CHUNKS"])))
    if os.environ.get("NTP_SYNC_KERNEL"):  # experiments: 1 LDG, 2 BULK 4x1, 3 BULK 3x2
        _lib.check(L.ntp_set_option(0, int(os.environ["NTP_SYNC_KERNEL"])))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        rows = sync_sweep_dist()
        if dist.get_rank() == 0:
            print(json.dumps({"device": torch.cuda.get_device_name(), "n_gpus": dist.get_world_size(),
                              f"sync_sweep_{dist.get_world_size()}gpu": rows}, indent=1))
        dist.destroy_process_group()
        return
    doc = {"device": torch.cuda.get_device_name(), "sync_sweep_1gpu": sync_sweep_local()}
    if not args.sync_only:
        doc["reconfig_8b_1gpu"] = reconfig(args.reconfig_layers)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
