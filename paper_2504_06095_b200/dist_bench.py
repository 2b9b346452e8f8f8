"""bench.py's N>1 arm: one process per GPU (torchrun), NVLink peer-memory sync.

The same workload as N=1 (gpt-1.3b, DP=2 TP4+TP3, bf16), with the 7 logical
ranks placed on the N GPUs by ``Placement.default`` (N>=8: one GPU per logical
rank, GPU 7 idle as the failed one; N=2: healthy replica on GPU 0, reduced on
GPU 1; N=4: 2+2 GPUs).  Each rank device-times its K steps with CUDA events;
rank 0 reports the max over ranks.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dist import NtpSyncGroup, Placement
from .workloads import SHAPES, pair_layout


def _max(x: float) -> float:
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run(args):
    from bench import (ELEM_BYTES, L2_BYTES, METRIC, W_H, W_R, WORKLOADS,  # noqa: I001 (repo root)
                       ClockSampler, peaks, workload_config)

    # NCCL warnings (and its version banner) go to stderr: bench.py keeps fd 1
    # pointed at stderr while this runs, so stdout is the one JSON line
    os.environ["NCCL_DEBUG"] = os.environ.get("NTP_NCCL_DEBUG", os.environ.get("NCCL_DEBUG", "WARN"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = int(os.environ.get("WORLD_SIZE", "1")) > torch.cuda.device_count()
    if shared:
        # more processes than GPUs (a functional run of an N-GPU placement on a
        # smaller box): processes share GPUs round-robin, host group over gloo
        # (NCCL puts at most one rank on a GPU); the timings are not N-GPU numbers
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    L = _lib.load()
    if os.environ.get("NTP_SYNC_KERNEL"):  # experiments: 1 LDG, 2 BULK, 3 BULK2
        _lib.check(L.ntp_set_option(0, int(os.environ["NTP_SYNC_KERNEL"])))
    shape = SHAPES[args.workload]
    n1, n2 = 4, 3
    lay = pair_layout(shape, n1, n2)
    plc = Placement.default(world, n1, n2)
    dt = WORKLOADS[args.workload][4]
    dtype, eb = {"bf16": torch.bfloat16, "f32": torch.float32}[dt], ELEM_BYTES[dt]
    nseg = len(shape.segments())
    pieces = [list(range(i * nseg, (i + 1) * nseg)) for i in range(lay.layers)]  # e2e: per layer
    grp = NtpSyncGroup(lay, plc, dtype, device=local, pieces=pieces).upload()
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    for s in grp.hosted:
        a = grp.arena(s)
        a.copy_(torch.randn(a.numel(), generator=gen, device="cuda").to(dtype))
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    dist.barrier()
    # small workloads would stay L2-resident between steps: flush (256 MB
    # write) before every timed step; the flushes are timed alone afterwards
    # and subtracted
    hosted_bytes = sum(grp.slot_elems[s] for s in grp.hosted) * eb
    flush = (torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
             if 2 * lay.elems * eb <= 2 * L2_BYTES else None)
    flush_fn = (lambda: flush.fill_(1)) if flush is not None else None  # noqa: E731
    use_graph = not getattr(args, "no_graph", False)

    def one():
        # one step as one CUDA-graph launch (recorded during warm-up): the
        # host's launch rate never paces the device (it would at small sizes)
        if use_graph:
            grp.step_graph(W_H, W_R, stream, prologue=flush_fn)
        else:
            if flush_fn is not None:
                flush_fn()
            grp.step(W_H, W_R, stream)

    for _ in range(max(args.warmup, 3)):
        one()
    torch.cuda.synchronize()
    dist.barrier()
    if grp.status() != 0:
        raise RuntimeError(f"rank {rank}: signal timeout during warm-up")
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    clocks.mark("t0")
    e0.record(stream)
    for _ in range(args.steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark("t1")
    dist.barrier()
    clk = clocks.stop()
    total_ms = e0.elapsed_time(e1)
    flush_ms = 0.0
    if flush is not None:
        for _ in range(3):
            flush_fn()
        e0.record(stream)
        for _ in range(args.steps):
            flush_fn()
        e1.record(stream)
        torch.cuda.synchronize()
        flush_ms = e0.elapsed_time(e1)
    ms = _max((total_ms - flush_ms) / args.steps)
    timing_detail = {"total_ms_rank0": round(total_ms, 4), "flush_ms_rank0": round(flush_ms, 4),
                     "total_ms_max": round(_max(total_ms), 4)}
    # NVLink bytes per launch: the committed ncu measurement of this placement's
    # per-process plans (NVML's NVLink throughput counters are not supported on
    # these boxes, and merely querying them slowed the step by 17 %: DESIGN.md 6)
    rec = _ncu_nvlink(args.workload, world)
    traffic = int(rec["busiest_direction_user_data_bytes"]) if rec else None
    traffic_raw = int(rec["busiest_direction_bytes"]) if rec else None
    traffic_src = ("ncu nvltx/nvlrx__bytes_data_user.sum of this placement's per-process plans "
                   "(scripts/nvlink_traffic.py, profiles/ncu_nvlink_traffic.json): payload bytes "
                   "in the busiest GPU direction; traffic_with_protocol adds NVLink packet "
                   "overhead (read requests, headers)" if rec else
                   "not measured for this workload / N")
    kernel_ms = ms
    if grp.status() != 0:
        raise RuntimeError(f"rank {rank}: signal timeout")
    S = lay.elems
    B = busiest_bytes_for(lay, plc, eb)
    pk = peaks()
    achieved = B / (ms * 1e-3) / 1e9
    out = None
    e2e = run_e2e(args, grp, lay, dtype, eb)
    check = None
    if getattr(args, "check", False):  # the checker lives in bench.py (it runs the oracle)
        from bench import check_dist  # noqa: I001
        check = check_dist(args, grp, lay, dtype, _max)
    if rank == 0:
        out = {"metric": METRIC, "value": round(S * eb / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
               "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
               "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": dt,
               "data": "synthetic (N(0,1) gradients)",
               "config": workload_config(args.workload, world),
               **({"shared_gpus": f"{world} processes on {torch.cuda.device_count()} GPUs: a "
                                  "functional run of the placement, not an N-GPU measurement"}
                  if shared else {}),
               "placement": {"healthy": list(plc.h_proc), "reduced": list(plc.r_proc),
                             "busiest_gpu_bytes_per_direction": B,
                             "hosted_bytes_rank0": hosted_bytes},
               "roofline": {"bound": "nvlink",
                            "kernel": f"ntp::plan_kernel_bulk<{dt},weighted,4,signaled>",
                            "achieved": round(achieved, 1), "peak": pk["nvlink_gbs"],
                            "peak_src": "measured peer copy 770 GB/s/direction (B200_PROFILING.md)",
                            "unit": "GB/s", "frac": round(achieved / pk["nvlink_gbs"], 4),
                            "algorithmic_bytes_per_launch": B, "traffic": traffic,
                            "traffic_src": traffic_src,
                            "traffic_with_protocol": traffic_raw,
                            "traffic_over_algorithmic": (round(traffic / B, 3) if traffic and B
                                                         else None),
                            "kernel_ms": round(kernel_ms, 4)},
               "timing": ("K steps, each one CUDA-graph launch" if use_graph else "K eager steps")
                         + (" after a 256 MB L2 flush; K flushes timed alone and subtracted"
                            if flush is not None else ""),
               "timing_detail": timing_detail,
               "gpu_launches": args.steps * _launches_per_step(grp),
               "clocks": clk, "e2e": e2e}
        if check is not None:
            out["check"] = check
    dist.barrier()
    grp.close()
    dist.barrier()
    dist.destroy_process_group()
    return out


def _ncu_nvlink(workload: str, world: int):
    """The committed ncu NVLink measurement for (workload, N), if any."""
    import json
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_nvlink_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    rec = d.get(workload, {}).get(str(world))
    if rec and "busiest_direction_bytes" in rec and "busiest_direction_user_data_bytes" in rec:
        return rec
    return None


def busiest_bytes_for(lay, plc: Placement, eb: int) -> int:
    """Busiest GPU's one-direction NVLink bytes for this placement: elements it
    hosts whose partner copy lives on another GPU."""
    worst = 0
    for rank in set(plc.h_proc) | set(plc.r_proc):
        remote = 0
        for k, unit, hc, rc, hb, rbase in lay.segs:
            comp = np.empty(k, dtype=np.int64)
            for r, c in enumerate(hc):
                comp[c] = r
            for j, c in enumerate(rc):
                hp = np.array(plc.h_proc)[comp[c]]
                rp = plc.r_proc[j]
                if rp == rank:
                    remote += int((hp != rank).sum()) * unit
                else:
                    remote += int(((hp == rank)).sum()) * unit
        worst = max(worst, remote)
    return worst * eb


def _launches_per_step(grp, plan="whole") -> int:
    """Kernels one step() launches on this rank (see NtpSyncGroup.step)."""
    p = grp.plan if plan == "whole" else plan
    if grp.partners and grp.fused_step:
        return 1
    return int(p is not None) + int(bool(grp.post_ready)) + int(bool(grp.wait_done))


def run_e2e(args, grp, lay, dtype, eb):
    """Per rank: pinned host arenas -> device, sync, device -> host; max over
    ranks.  Pipelined per layer (the group's pieces): the H2D of layer i+1, the
    peer-memory sync of layer i and the D2H of layer i-1 run at once on three
    streams, so a step is bound by the host link's two directions."""
    from bench import W_H, W_R  # noqa: I001
    host = {s: torch.empty(grp.slot_elems[s], dtype=dtype).pin_memory() for s in grp.hosted}
    dev = {s: grp.arena(s) for s in grp.hosted}
    stream = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    steps = max(2, min(args.e2e_steps, args.steps))
    ranges = [grp.piece_ranges(i) for i in range(len(grp.pieces))]

    prev = [None]  # per piece: the previous step's D2H of that piece

    def one(sync=True):
        # piece i's H2D waits only for the previous step's D2H of piece i, so
        # back-to-back steps keep both host-link directions busy
        if prev[0] is None:
            h2d_s.wait_stream(stream)
        done = []
        for i, rg in enumerate(ranges):
            if prev[0] is not None:
                h2d_s.wait_event(prev[0][i])
            with torch.cuda.stream(h2d_s):
                for s, (lo, hi) in rg.items():
                    dev[s][lo:hi].copy_(host[s][lo:hi], non_blocking=True)
            stream.wait_stream(h2d_s)
            if sync:
                grp.step(W_H, W_R, stream, piece=i)
            d2h_s.wait_stream(stream)
            with torch.cuda.stream(d2h_s):
                for s, (lo, hi) in rg.items():
                    host[s][lo:hi].copy_(dev[s][lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(d2h_s)
            done.append(ev)
        prev[0] = done
        stream.wait_stream(d2h_s)

    one()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = _max(e0.elapsed_time(e1) / steps)
    wall_ms = (time.perf_counter() - t0) * 1e3 / steps
    # host-link bound at this N: the same pipelined copies with no sync, every
    # rank at once (ranks may share host bridges / memory)
    one(sync=False)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(2):
        one(sync=False)
    e1.record(stream)
    torch.cuda.synchronize()
    copy_ms = _max(e0.elapsed_time(e1) / 2)
    nbytes = sum(grp.slot_elems[s] for s in grp.hosted) * eb
    h2d = int(_max(float(nbytes)))
    return {"value": round(lay.elems * eb / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(ms, 3), "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d,
            "note": "per-rank max; every rank copies its own arenas over its own PCIe link, "
                    "pipelined per layer (H2D / peer sync / D2H on three streams)",
            "pipeline_pieces": len(ranges),
            "host_copies_only_ms": round(copy_ms, 3),
            "host_link_frac": round(copy_ms / ms, 3),
            "gpu_launches_per_step": sum(_launches_per_step(grp, p) for p in grp.piece_plans),
            "wall_ms_per_step": round(wall_ms, 3)}
