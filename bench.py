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


def cpu_sample(shape, n1, n2, layers=1, threads=None, reps=3, seed=0, passes=1):
    """Time oracle.nonuniform_sync (fp64, the reference's arithmetic) on `layers`
    layers of the workload, `passes` times over the same host buffers (so a
    whole multi-layer step can be timed with one layer's memory); returns
    (seconds per pass set, best of reps; elements per pass; threads)."""
    from oracle import oracle as O
    from paper_2504_06095_b200.workloads import pair_layout
    if threads:
        O.set_threads(threads)
    lay = pair_layout(shape, n1, n2, layers=layers)
    rng = np.random.default_rng(seed)
    best = float("inf")
    hb = [rng.standard_normal(e) for e in lay.h_elems]
    rb = [rng.standard_normal(e) for e in lay.r_elems]
    for _ in range(reps):
        t = 0.0
        for k, unit, hc, rc, h_base, r_base in lay.segs:
            # per-segment views into the rank arenas (unit-major)
            hv = [np.ascontiguousarray(b[s:s + len(c) * unit]) for b, c, s in zip(hb, hc, h_base)]
            rv = [np.ascontiguousarray(b[s:s + len(c) * unit]) for b, c, s in zip(rb, rc, r_base)]
            smap_comp = np.empty(k, dtype=np.int64)
            smap_sync = np.empty(k, dtype=np.int64)
            for r, c in enumerate(hc):
                smap_comp[c] = r
            for r, c in enumerate(rc):
                smap_sync[c] = r
            for _ in range(passes):
                t0 = time.perf_counter()
                O.nonuniform_sync(smap_comp, smap_sync, hc, rc, hv, rv, unit, op=O.OP_WEIGHTED,
                                  weights=(W_H, W_R))
                t += time.perf_counter() - t0
        best = min(best, t)
    return best, lay.elems, O.num_threads()


# ---------------------------------------------------------------------------
# our arm, one GPU


def run_single(args):
    import torch
    from paper_2504_06095_b200 import _lib
    from paper_2504_06095_b200.plans import OPS, tensor_ptrs
    from paper_2504_06095_b200.workloads import SHAPES, build_plan, pair_layout

    _lib.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    shape = SHAPES[args.workload]
    dtype = torch.bfloat16
    eb = 2
    lay = pair_layout(shape, 4, 3)
    plan = build_plan(lay, dtype).upload(0)
    gen = torch.Generator(device=dev).manual_seed(0)
    arenas = [torch.randn(e, generator=gen, device=dev, dtype=torch.float32).to(dtype)
              for e in lay.h_elems + lay.r_elems]
    ptrs = tensor_ptrs(arenas)
    S = lay.elems
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.grad_sync(ptrs, OPS["weighted"], W_H, W_R, stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    clocks.mark("t0")
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark("t1")
    ms_total = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms = ms_total / args.steps
    value = S * eb / (ms * 1e-3) / 1e9
    pk = peaks()
    hbm_bytes = 4 * S * eb  # read both replicas, write both
    achieved = hbm_bytes / (ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": "ntp::plan_kernel_bulk<bf16,weighted,4>",
            "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "peak_src": pk["src"],
            "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "algorithmic_bytes_per_launch": hbm_bytes, "traffic": _ncu_traffic()}
    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
           "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (N(0,1) bf16 gradients, torch.Generator seed 0)",
           "config": {"workload": f"{shape.name} DP=2 TP4+TP3 full-step grad sync "
                                  "(BASELINE configs[1]), 7 logical ranks on 1 GPU",
                      "layers": shape.layers, "hidden": shape.hidden, "ffn": shape.ffn,
                      "heads": shape.heads, "grad_bytes_per_replica": S * eb,
                      "weights": [round(W_H, 6), round(W_R, 6)],
                      "l2": "inputs 4.8 GB >> 126 MB L2 (no flush needed)",
                      "plan_chunks": plan.stats["n_chunks"]},
           "roofline": roof, "gpu_launches": args.steps, "clocks": clk}
    if not args.no_e2e:
        out["e2e"] = run_e2e_single(args, lay, plan, dtype, eb)
    if not args.no_cpu:
        # one whole step of the workload: all layers synced in turn through one
        # layer's host buffers (memory stays at one layer), best of 8 (~10 s)
        t, elems, thr = cpu_sample(shape, 4, 3, layers=1, passes=shape.layers, reps=8)
        out["cpu_baseline"] = {"value": round(shape.layers * elems * eb / t / 1e9, 3),
                               "unit": "GB/s", "cores": thr, "kind": "port",
                               "sample": f"one full step: {shape.layers} layers x {elems} elements "
                                         "per replica, each layer through the same host buffers; "
                                         "oracle fp64 3-step nonuniform_grad_sync, best of 8 steps",
                               "seconds_per_step": round(t, 3)}
    return out


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
                                           segs_per_piece=spp))
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


def _ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


# ---------------------------------------------------------------------------
# reference arm: the oracle port of the reference's CPU path, all host threads


def run_reference(args):
    from paper_2504_06095_b200.workloads import SHAPES
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    shape = SHAPES[args.workload]
    eb = 2
    times = []
    for i in range(max(args.warmup, 0) + args.steps):
        t, elems, thr = cpu_sample(shape, 4, 3, layers=1, reps=1, seed=i)
        if i >= args.warmup:
            times.append(t)
    ms = 1e3 * float(np.mean(times))
    value = elems * eb / (ms * 1e-3) / 1e9
    return {"metric": METRIC, "impl": "reference", "value": round(value, 3), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (N(0,1))",
            "config": {"workload": f"{shape.name} DP=2 TP4+TP3 grad sync, 1-layer sample per step"},
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": thr, "kind": "port",
                             "sample": f"1 of {shape.layers} layers ({elems} elements per replica) "
                                       "per step; oracle/ntp_oracle.c restatement of "
                                       "tpnumerics.py:289-356 (the reference is pure Python; "
                                       "its 405 ms C1 time is in BASELINE.md)"},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


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
    args = ap.parse_args(argv)
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return 0
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
