#!/usr/bin/env python
"""Benchmark of the NTP gradient reshard-and-reduce (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One *step* = one nonuniform gradient sync of the whole synthetic workload:
every unit of the healthy TP4 replica's gradient and the degraded TP3
replica's gradient is reduced (weights = local batch share 4/7, 3/7) and
written back to both replicas' layouts.

N=1 workload: BASELINE.json configs[1], GPT-style 1.3B (24 layers, hidden
2048, ffn 8192, 16 heads), bf16, DP=2 TP4+TP3 -- all 7 logical ranks' gradient
arenas on one B200 (HBM-bound; inputs 4.8 GB >> 126 MB L2, so no L2 flush is
needed between steps).  N>1: one process per GPU (torchrun), see
paper_2504_06095_b200/dist.py; the reduced replica's GPUs pull/push peers'
units over NVLink.

value = synchronized gradient bytes per second = (elements of one replica's
gradient x 2 bytes) / device time per step, max over ranks.  ``roofline``
reports the dominant kernel against its bound (HBM at N=1: 4*S*b bytes per
launch; NVLink at N>1: the busiest GPU's one-direction bytes).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NTP grad-sync GB/s & % NVLink roofline (device-timed, max over ranks) vs CPU ref"
W_H, W_R = 4.0 / 7.0, 3.0 / 7.0  # local-batch share of TP4 (lb 4) and TP3 (lb 3) replicas
L2_BYTES = 126 << 20

# BASELINE.json configs, restated here so the reference arm needs no product
# import (tests/test_bench_contract.py checks they equal workloads.SHAPES)
WORKLOADS = {
    # name: (hidden, ffn, heads, layers, dtype, BASELINE.json config)
    "gpt-1.3b": (2048, 8192, 16, 24, "bf16", "configs[1]"),
    "llama3-8b-shaped": (4096, 14336, 32, 32, "bf16", "configs[3]"),
    "mlp-h1024-ffn4096": (1024, 4096, 0, 1, "f32", "configs[0]"),
}
ELEM_BYTES = {"bf16": 2, "f32": 4}


def workload_elems(name: str) -> int:
    """Elements of one replica's gradient (every layer, MLP + attention units)."""
    hidden, ffn, heads, layers = WORKLOADS[name][:4]
    per = ffn * 2 * hidden + (heads * 4 * hidden * (hidden // heads) if heads else 0)
    return layers * per


def workload_config(name: str, n_gpus: int) -> dict:
    """The `config` object both arms print (identical, so the driver can pair them)."""
    hidden, ffn, heads, layers, dt, which = WORKLOADS[name]
    S = workload_elems(name)
    eb = ELEM_BYTES[dt]
    l2 = ("inputs %.1f GB >> 126 MB L2 (no flush needed)" % (2 * S * eb / 1e9)
          if 2 * S * eb > 2 * L2_BYTES else
          "inputs %.0f MB < 2x L2: L2 flushed (256 MB write) before every timed step"
          % (2 * S * eb / 1e6))
    return {"workload": f"{name} DP=2 TP4+TP3 full-step grad sync (BASELINE {which}), "
                        f"{'7 logical ranks on 1 GPU' if n_gpus == 1 else 'logical ranks over %d GPUs' % n_gpus}",
            "layers": layers, "hidden": hidden, "ffn": ffn, "heads": heads,
            "grad_bytes_per_replica": S * eb, "weights": [round(W_H, 6), round(W_R, 6)],
            "l2": l2}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured", "nvlink_gbs": 770.0}
    return {"hbm_gbs": 6650.0, "src": "fallback", "nvlink_gbs": 770.0}


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            time.sleep(0.5)  # let nvidia-smi attach before the timed region
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, which):
        setattr(self, which, time.time())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [l for t, l in self.lines if self.t0 is not None and self.t0 - 0.06 <= t <= self.t1 + 0.06]
        if not rows:
            rows = [l for _, l in self.lines]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [p.strip() for p in r.split(",")]
            if len(parts) < 10:
                continue
            try:
                sm.append(float(parts[2]))
                smax.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[6:10]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement of the reference's nonuniform_grad_sync


def cpu_sample(name, n1=4, n2=3, layers=1, threads=None, reps=3, seed=0, passes=1):
    """Time oracle.nonuniform_sync (fp64, the reference's arithmetic) on `layers`
    layers of workload `name`, `passes` times over the same host buffers (so a
    whole multi-layer step is timed with one layer's memory: every layer has
    the same shard maps and sizes); returns (seconds for one pass set, best of
    reps; elements per pass; threads).  Only oracle/ is used: no product code
    runs or loads on this leg."""
    from oracle import oracle as O
    if threads:
        O.set_threads(threads)
    hidden, ffn, heads = WORKLOADS[name][:3]
    segs, h_elems, r_elems = O.pair_layout(hidden, ffn, heads, layers, n1, n2)
    rng = np.random.default_rng(seed)
    best = float("inf")
    hb = [rng.standard_normal(e) for e in h_elems]
    rb = [rng.standard_normal(e) for e in r_elems]
    # per-segment contiguous views into the rank arenas (unit-major)
    views = [O.segment_views(seg, hb, rb) for seg in segs]
    for _ in range(reps):
        t = 0.0
        for _ in range(passes):
            t0 = time.perf_counter()
            for seg, (hv, rv) in zip(segs, views):
                O.nonuniform_sync(seg[2], seg[3], seg[4], seg[5], hv, rv, seg[1],
                                  op=O.OP_WEIGHTED, weights=(W_H, W_R))
            t += time.perf_counter() - t0
        best = min(best, t)
    return best, sum(h_elems), O.num_threads()


# ---------------------------------------------------------------------------
# our arm, one GPU


def _torch_dtype(name):
    import torch
    return {"bf16": torch.bfloat16, "f32": torch.float32}[WORKLOADS[name][4]]


def run_single(args):
    import torch
    from paper_2504_06095_b200 import _lib
    from paper_2504_06095_b200.plans import OPS, tensor_ptrs
    from paper_2504_06095_b200.workloads import SHAPES, build_plan, pair_layout

    _lib.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    shape = SHAPES[args.workload]
    dtype = _torch_dtype(args.workload)
    eb = ELEM_BYTES[WORKLOADS[args.workload][4]]
    lay = pair_layout(shape, 4, 3)
    plan = build_plan(lay, dtype).upload(0)
    gen = torch.Generator(device=dev).manual_seed(0)
    arenas = [torch.randn(e, generator=gen, device=dev, dtype=torch.float32).to(dtype)
              for e in lay.h_elems + lay.r_elems]
    ptrs = tensor_ptrs(arenas)
    S = lay.elems
    stream = torch.cuda.current_stream(dev)
    flush = None
    if 2 * S * eb <= 2 * L2_BYTES:  # inputs could stay L2-resident: flush before each step
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        plan.grad_sync(ptrs, OPS["weighted"], W_H, W_R, stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * (args.steps if flush is not None else 1))]
    torch.cuda.synchronize()
    clocks.mark("t0")
    if flush is None:
        ev[0].record(stream)
        for _ in range(args.steps):
            step()
        ev[1].record(stream)
    else:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[2 * i].record(stream)
            step()
            ev[2 * i + 1].record(stream)
    torch.cuda.synchronize()
    clocks.mark("t1")
    ms_total = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(len(ev) // 2))
    clk = clocks.stop()
    ms = ms_total / args.steps
    value = S * eb / (ms * 1e-3) / 1e9
    pk = peaks()
    hbm_bytes = 4 * S * eb  # read both replicas, write both
    achieved = hbm_bytes / (ms * 1e-3) / 1e9
    kname = "ntp::plan_kernel_%s<%s,weighted>" % (
        "bulk" if plan.stats["n_chunks"] >= 4 * 148 else "vec", WORKLOADS[args.workload][4])
    roof = {"bound": "hbm", "kernel": kname,
            "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "peak_src": pk["src"],
            "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "algorithmic_bytes_per_launch": hbm_bytes,
            "traffic": _ncu_traffic(args.workload)}
    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
           "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": WORKLOADS[args.workload][4],
           "data": "synthetic (N(0,1) gradients, torch.Generator seed 0)",
           "config": workload_config(args.workload, 1),
           "plan": {"chunks": plan.stats["n_chunks"], "table_bytes": 16 * plan.stats["n_chunks"]},
           "roofline": roof, "gpu_launches": args.steps, "clocks": clk}
    if args.check:
        out["check"] = check_single(args, lay, plan, arenas, dtype)
    if not args.no_e2e:
        out["e2e"] = run_e2e_single(args, lay, plan, dtype, eb)
        if shape.layers == 1 and not shape.heads:
            out["e2e_reference_objects"] = run_e2e_reference_objects(args)
    if not args.no_cpu:
        # one whole step of the workload: all layers synced in turn through one
        # layer's host buffers (memory stays at one layer), best of a few (~10 s)
        reps = 8 if shape.layers > 1 else 40
        t, elems, thr = cpu_sample(args.workload, 4, 3, layers=1, passes=shape.layers, reps=reps)
        out["cpu_baseline"] = {"value": round(shape.layers * elems * eb / t / 1e9, 3),
                               "unit": "GB/s", "cores": thr, "kind": "port",
                               "sample": f"one full step: {shape.layers} layer(s) x {elems} elements "
                                         "per replica, each layer through the same host buffers; "
                                         "oracle fp64 3-step nonuniform_grad_sync, "
                                         f"best of {reps} steps",
                               "seconds_per_step": round(t, 4)}
    return out


def check_single(args, lay, plan, arenas, dtype):
    """--check: one more step on fresh inputs, every segment of every layer
    against the fp64 oracle."""
    hidden, ffn, heads, layers = WORKLOADS[args.workload][:4]
    return check_pair_arenas(hidden, ffn, heads, layers, plan, arenas, dtype, lay.h_elems,
                             lay.r_elems)


def check_pair_arenas(hidden, ffn, heads, layers, plan, arenas, dtype, h_elems, r_elems,
                      seed=12345, weights=(W_H, W_R), n1=4, n2=3):
    """Fill the 1-GPU arenas with fresh N(0,1) values, run ONE sync through
    `plan`, then compare every segment of every layer with the fp64 oracle on
    the same dtype-rounded inputs (streamed segment by segment).  The layout
    used to slice the arenas comes from the oracle's own shard map, and must
    equal the product's.  Returns a summary; raises when a segment is off."""
    import torch
    from oracle import oracle as O
    from paper_2504_06095_b200.plans import OPS, tensor_ptrs
    segs, oh, orr = O.pair_layout(hidden, ffn, heads, layers, n1, n2)
    if oh != list(h_elems) or orr != list(r_elems):
        raise RuntimeError("product arena layout differs from the oracle's")
    gen = torch.Generator(device=arenas[0].device).manual_seed(seed)
    for a in arenas:
        a.copy_(torch.randn(a.numel(), generator=gen, device=a.device).to(dtype))
    before = [a.cpu() for a in arenas]
    plan.grad_sync(tensor_ptrs(arenas), OPS["weighted"], weights[0], weights[1])
    torch.cuda.synchronize()
    after = [a.cpu() for a in arenas]
    worst, identical, t0 = 0.0, True, time.perf_counter()
    tol = {torch.bfloat16: 2e-2, torch.float16: 2e-3, torch.float32: 1e-6}[dtype]
    errs = []

    def f64(views):
        return [v.double().numpy() for v in views]
    for seg in segs:
        hv_in, rv_in = O.segment_views(seg, before[:n1], before[n1:])
        hv_out, rv_out = O.segment_views(seg, after[:n1], after[n1:])
        err, same = O.check_pair_segment(seg, f64(hv_in), f64(rv_in), f64(hv_out), f64(rv_out),
                                         weights)
        errs.append(err)
        worst = max(worst, err)
        identical &= same
    ok = worst <= tol and identical
    res = {"ok": ok, "segments": len(segs), "max_rel_err": worst, "tol": tol,
           "replicas_bit_identical": identical, "chunks": plan.stats["n_chunks"],
           "seconds": round(time.perf_counter() - t0, 1),
           "oracle": "oracle.nonuniform_sync fp64 (tpnumerics.py:289-356) on the same rounded inputs"}
    if not ok:
        bad = [i for i, e in enumerate(errs) if e > tol]
        raise RuntimeError(f"parity check failed: {res}, segments over tol: {bad[:10]}")
    return res


def _segment_input(slot: int, seg: int, n: int, dtype):
    """Deterministic N(0,1) input of one logical rank's slice of one segment
    (CPU, any process can regenerate any slot's values)."""
    import torch
    g = torch.Generator().manual_seed(1_000_003 * (slot + 1) + seg)
    return torch.randn(n, generator=g).to(dtype)


def check_dist(args, grp, lay, dtype, _max):
    """--check at N>1: the exact bench plans, every segment of every layer vs
    the fp64 oracle.  Every arena is refilled with per-(slot, segment) seeded
    values, ONE step runs, and each process checks the slots it hosts: it
    regenerates every slot's inputs of a segment on the CPU, runs the oracle's
    nonuniform_grad_sync (tpnumerics.py:289-356) and compares its own device
    outputs (Frobenius per segment).  Max over processes."""
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    rank = dist.get_rank()
    hidden, ffn, heads = lay.shape.hidden, lay.shape.ffn, lay.shape.heads
    segs, _, _ = O.pair_layout(hidden, ffn, heads, lay.layers, lay.n1, lay.n2)
    n1 = lay.n1
    nslots = n1 + lay.n2

    def slot_range(seg, s):
        k, unit, comp, sync, hc, rc, hb, rb = seg
        cols, base = (hc[s], hb[s]) if s < n1 else (rc[s - n1], rb[s - n1])
        return int(base), int(base) + len(cols) * unit
    for i, seg in enumerate(segs):
        for s in grp.hosted:
            lo, hi = slot_range(seg, s)
            grp.arena(s)[lo:hi].copy_(_segment_input(s, i, hi - lo, dtype))
    torch.cuda.synchronize()
    dist.barrier()
    grp.step(W_H, W_R)
    torch.cuda.synchronize()
    dist.barrier()
    worst, t0 = 0.0, time.perf_counter()
    for i, seg in enumerate(segs):
        if not grp.hosted:
            break
        ins = [_segment_input(s, i, slot_range(seg, s)[1] - slot_range(seg, s)[0], dtype)
               .double().numpy() for s in range(nslots)]
        k, unit, comp, sync, hc, rc, hb, rb = seg
        hw, rw = ins[:n1], ins[n1:]
        O.nonuniform_sync(comp, sync, hc, rc, hw, rw, unit, op=O.OP_WEIGHTED, weights=(W_H, W_R))
        want = hw + rw
        for s in grp.hosted:
            lo, hi = slot_range(seg, s)
            got = grp.arena(s)[lo:hi].double().cpu().numpy()
            worst = max(worst, O.rel_err(got, want[s]))
    worst = _max(worst)
    tol = {torch.bfloat16: 2e-2, torch.float32: 1e-6}[dtype]
    res = {"ok": worst <= tol, "segments": len(segs), "max_rel_err": worst, "tol": tol,
           "seconds": round(_max(time.perf_counter() - t0), 1),
           "oracle": "oracle.nonuniform_sync fp64 on the same rounded inputs; every process "
                     "checks the logical ranks it hosts"}
    if not res["ok"]:
        raise RuntimeError(f"bench --check failed at N={dist.get_world_size()}: {res} (rank {rank})")
    return res


def run_e2e_single(args, lay, plan, dtype, eb):
    """Same metric through the public host-buffer API: pinned host arenas in,
    H2D + sync + D2H inside the timed region."""
    import torch
    from paper_2504_06095_b200.hostsync import HostSync
    from paper_2504_06095_b200.workloads import layer_pieces
    lpp = int(os.environ.get("NTP_E2E_LAYERS_PER_PIECE", "1"))
    spp = int(os.environ.get("NTP_E2E_SEGS_PER_PIECE", "0")) or None
    hs = HostSync(plan, [e for e in lay.h_elems + lay.r_elems], dtype, device=0,
                  piece_plans=layer_pieces(lay, dtype, 0, layers_per_piece=lpp,
                                           segs_per_piece=spp),
                  back_to_back=True)  # the timed loop re-runs the same host buffers
    gen = torch.Generator().manual_seed(1)
    host = [torch.randn(e, generator=gen, dtype=torch.float32).to(dtype).pin_memory()
            for e in lay.h_elems + lay.r_elems]
    # host-link context: one direction alone, the same bytes as a step's H2D
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for d, h in zip(hs.arenas, host):
        d.copy_(h, non_blocking=True)
    s1.record()
    torch.cuda.synchronize()
    h2d_gbs = sum(h.numel() for h in host) * eb / (s0.elapsed_time(s1) * 1e-3) / 1e9
    # and both directions at once (what a pipelined step needs): 2 GiB each way
    # in 8 pieces per direction on two streams, like the pipeline's copies,
    # between device scratch and pinned host scratch
    n, pieces = 2 << 30, 8
    hs_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    hs_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    dv = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    step = n // pieces
    best = float("inf")
    for _ in range(4):  # first pass warms the pinned pages; best of the rest
        torch.cuda.synchronize()
        s0.record()
        sa.wait_stream(torch.cuda.current_stream())
        sb.wait_stream(torch.cuda.current_stream())
        for i in range(pieces):
            lo, hi = i * step, (i + 1) * step
            with torch.cuda.stream(sa):
                dv[lo:hi].copy_(hs_in[lo:hi], non_blocking=True)
            with torch.cuda.stream(sb):
                hs_out[lo:hi].copy_(dv[n + lo:n + hi], non_blocking=True)
        torch.cuda.current_stream().wait_stream(sa)
        torch.cuda.current_stream().wait_stream(sb)
        s1.record()
        torch.cuda.synchronize()
        best = min(best, s0.elapsed_time(s1))
    duplex_gbs = n / (best * 1e-3) / 1e9
    del hs_in, hs_out, dv
    steps = max(2, min(args.e2e_steps, args.steps))
    for _ in range(2):
        hs.run(host, W_H, W_R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        hs.run(host, W_H, W_R)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nbytes = sum(lay.h_elems + lay.r_elems) * eb
    return {"value": round(lay.elems * eb / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(ms, 3), "steps": steps,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "wall_ms_per_step": round((time.perf_counter() - t0) * 1e3 / steps, 3),
            "gpu_launches_per_step": hs.launches_per_run,
            "pipeline_pieces": len(hs.pieces or []),
            "host_link_h2d_only_gbs": round(h2d_gbs, 1),
            "host_link_duplex_gbs_per_direction": round(duplex_gbs, 1),
            "host_link_bound_ms": round(nbytes / (duplex_gbs * 1e9) * 1e3, 2),
            "host_link_frac": round(nbytes / (duplex_gbs * 1e9) * 1e3 / ms, 3)}


def run_e2e_reference_objects(args, reps=20):
    """C1 through the reference's own call: tpnumerics.nonuniform_grad_sync on
    replica objects shaped like ntpsim's MlpReplica (numpy fp64 grad_a [h, n_r]
    / grad_b [n_r, h] lists, mutated in place; tpnumerics.py:131-155,
    289-356).  The product's host path stages them into pinned unit-major
    buffers, runs the fp64 kernel and writes the results back (plan and
    staging cached after the first call); wall time per call."""
    import torch
    from types import SimpleNamespace
    from paper_2504_06095_b200 import tpnumerics as T
    from paper_2504_06095_b200.shardmap import build_shard_map
    hidden, ffn = WORKLOADS[args.workload][:2]
    smap = build_shard_map(ffn, 4, 3)
    rng = np.random.default_rng(0)
    layer = T.MlpLayer(np.zeros((hidden, ffn)), np.zeros((ffn, hidden)))

    def replica(cols):
        return SimpleNamespace(layer=layer, n=len(cols), cols=cols,
                               grad_a=[rng.standard_normal((hidden, len(c))) for c in cols],
                               grad_b=[rng.standard_normal((len(c), hidden)) for c in cols])
    h, r = replica(T.assignment_from_comp(smap)), replica(T.assignment_from_sync(smap))
    T.nonuniform_grad_sync(h, r, smap, weights=(W_H, W_R))  # builds and caches plan + staging
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        T.nonuniform_grad_sync(h, r, smap, weights=(W_H, W_R))
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    elems = ffn * 2 * hidden
    return {"value": round(elems * 8 / t / 1e9, 3), "unit": "GB/s", "dtype": "f64",
            "ms_per_call_median": round(t * 1e3, 3), "calls": reps,
            "h2d_bytes_per_step": 2 * elems * 8, "d2h_bytes_per_step": 2 * elems * 8,
            "note": "wall time of tpnumerics.nonuniform_grad_sync on ntpsim-shaped numpy "
                    "replicas (fp64, in place): host restaging + H2D + kernel + D2H; the "
                    "reference's own Python call takes 405 ms on this shape (BASELINE.md)"}


def _ncu_traffic(workload):
    """DRAM bytes per launch of the bench kernel from the committed ncu --set
    full capture (profiles/ncu_traffic.json, keyed by workload)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        rec = d.get(workload)
        if rec:
            return rec.get("dram_bytes_per_launch")
    return None


# ---------------------------------------------------------------------------
# reference arm: the oracle port of the reference's CPU path, all host threads


def run_reference(args):
    """The reference's CPU path (the oracle's C restatement of
    tpnumerics.py:289-356, fp64, every host thread) on the SAME workload and
    config as our arm: each timed step syncs every layer of the workload.  Only
    oracle/ runs here (the product library is never imported or loaded)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    name = args.workload
    layers = WORKLOADS[name][3]
    eb = ELEM_BYTES[WORKLOADS[name][4]]
    times = []
    thr = 0
    elems = 0
    for i in range(max(args.warmup, 0) + args.steps):
        t, elems, thr = cpu_sample(name, 4, 3, layers=1, passes=layers, reps=1, seed=i)
        if i >= args.warmup:
            times.append(t)
    ms = 1e3 * float(np.mean(times))
    S = layers * elems
    assert S == workload_elems(name)
    value = S * eb / (ms * 1e-3) / 1e9
    sample = (f"every step = the whole workload: {layers} layer(s) x {elems} elements per "
              "replica, synced layer by layer through one layer's host buffers (same shard maps "
              "and sizes as every layer); oracle/ntp_oracle.c fp64 restatement of "
              "tpnumerics.py:289-356 (the reference is pure Python; its 405 ms C1 time is in "
              "BASELINE.md)")
    return {"metric": METRIC, "impl": "reference", "value": round(value, 3), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (N(0,1))",
            "config": workload_config(name, args.gpus),
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": thr, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _reexec_torchrun(args, argv):
    """`python bench.py --gpus N` (N>1) outside torchrun: relaunch this script
    under torch.distributed.run with one process per GPU (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="gpt-1.3b")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N>1: launch every step eagerly instead of as one CUDA-graph launch")
    ap.add_argument("--check", action="store_true",
                    help="after the timed region, check every segment of one more step "
                         "against the fp64 oracle")
    args = ap.parse_args(argv)
    if args.workload not in WORKLOADS:
        ap.error(f"--workload must be one of {sorted(WORKLOADS)}")
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _reexec_torchrun(args, sys.argv[1:] if argv is None else argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    with _stdout_to_stderr():  # library banners (NCCL's version line) stay off stdout
        if world > 1 or args.gpus > 1:
            from paper_2504_06095_b200 import dist_bench
            out = dist_bench.run(args)
        else:
            out = run_single(args)
    if out is not None:
        print(json.dumps(out), flush=True)
    return 0


class _stdout_to_stderr:
    """Point fd 1 at stderr while the benchmark runs, so the only thing on
    stdout is the JSON line printed after it (NCCL prints its version banner
    with printf at NCCL_DEBUG=WARN/VERSION)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        try:
            import ctypes
            ctypes.CDLL(None).fflush(None)
        except OSError:
            pass
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


if __name__ == "__main__":
    sys.exit(main())
