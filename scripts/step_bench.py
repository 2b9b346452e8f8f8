"""Degraded-replica step overhead (north_star: <= 5 % over uniform TP).

One process per GPU (torchrun).  Two DP replicas of an L-layer MLP stack
(hidden h, ffn k; the reference's 2-matrix GeLU MLP, tpnumerics.py:177-252):

  * NTP run:      healthy TP-n1 + degraded TP-n2 (local batch scaled by n2/n1,
                  so every GPU does the same GEMM work; policy.py:139-148 shrinks
                  the reduced replica's batch the same way)
  * uniform run:  healthy TP-n1 + healthy TP-n1

Per layer, in reverse order, every GPU runs its shard's backward on the tensor
cores (D = (G B^T) * GeLU'(H); dB = Y^T G and dA^T = D^T X written straight
into the layer's unit-major gradient arena), then that layer's gradient sync
(dist.NtpSyncGroup: NVLink peer-memory reduce, weights = local batch shares)
is launched on a side stream so it overlaps the next layer's GEMMs.

Reported per run (device time, max over ranks): backward alone, sync alone,
backward + overlapped sync.  overhead = step(NTP) / step(uniform) - 1.

    torchrun --nproc-per-node 4 scripts/step_bench.py [--layers 8 --tokens 8192]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.linear import MlpShard  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_config(args, n1, n2, local):
    rank = dist.get_rank()
    h, k, L = args.hidden, args.ffn, args.layers
    shape = ModelShape("step", h, k, 0, 1)
    lay = pair_layout(shape, n1, n2)
    plc = Placement.default(dist.get_world_size(), n1, n2)
    tok_h = args.tokens
    tok_r = args.tokens * n2 // n1
    w_h, w_r = tok_h / (tok_h + tok_r), tok_r / (tok_h + tok_r)
    groups = [NtpSyncGroup(lay, plc, torch.bfloat16, local).upload() for _ in range(L)]
    staging = [NtpSyncGroup(lay, plc, torch.bfloat16, local).upload() for _ in range(L)]
    g = torch.Generator(device="cuda").manual_seed(rank)
    rng = np.random.default_rng(rank)
    shards = []   # per layer: [(shard, X, G, grads_view)]
    Xh = torch.randn((tok_h, h), generator=g, device="cuda").to(torch.bfloat16)
    Gh = torch.randn((tok_h, h), generator=g, device="cuda").to(torch.bfloat16)
    Xr = torch.randn((tok_r, h), generator=g, device="cuda").to(torch.bfloat16)
    Gr = torch.randn((tok_r, h), generator=g, device="cuda").to(torch.bfloat16)
    A = rng.standard_normal((h, k)) / np.sqrt(h)
    B = rng.standard_normal((k, h)) / np.sqrt(k)
    k_seg, unit, hc, rc, hb, rb = lay.segs[0]
    for li in range(L):
        per = []
        for s in groups[li].hosted:
            healthy = s < n1
            cols = hc[s] if healthy else rc[s - n1]
            sh = MlpShard(A, B, cols)
            X, G = (Xh, Gh) if healthy else (Xr, Gr)
            Z = torch.empty((X.shape[0], h), dtype=torch.float32, device="cuda")
            sh.forward(X, Z)  # H, Y for the backward
            grads = groups[li].arena(s).view(len(cols), 2, h)
            per.append((sh, X, G, grads))
        shards.append(per)
    torch.cuda.synchronize()
    dist.barrier()
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=-1)  # sync CTAs are scheduled ahead of GEMM CTAs

    def backward(overlap: bool, sync: bool = True):
        for li in reversed(range(L)):
            for sh, X, G, grads in shards[li]:
                sh.backward(X, G, grads)
            if sync and overlap:
                ev = torch.cuda.Event()
                ev.record(main)
                side.wait_event(ev)
                groups[li].step(w_h, w_r, side)
        if sync and not overlap:
            for li in reversed(range(L)):
                groups[li].step(w_h, w_r, main)
        main.wait_stream(side)

    def sync_only():
        for li in reversed(range(L)):
            groups[li].step(w_h, w_r, main)

    def timeline():
        """One overlapped backward with events: per layer, when its GEMMs and its
        sync finished (ms from the start), on this rank."""
        t0 = torch.cuda.Event(enable_timing=True)
        g_end, s_end = [], []
        torch.cuda.synchronize()
        dist.barrier()
        t0.record(main)
        for li in reversed(range(L)):
            for sh, X, G, grads in shards[li]:
                sh.backward(X, G, grads)
            e = torch.cuda.Event(enable_timing=True)
            e.record(main)
            g_end.append(e)
            side.wait_event(e)
            groups[li].step(w_h, w_r, side)
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record(side)
            s_end.append(e2)
        main.wait_stream(side)
        torch.cuda.synchronize()
        return {"gemm_done_ms": [round(t0.elapsed_time(e), 3) for e in g_end],
                "sync_done_ms": [round(t0.elapsed_time(e), 3) for e in s_end]}

    # fused wgrad + sync: every GPU's wgrad epilogue red.adds its weighted
    # gradient into its own arena and the partner replica's (zeroed first)
    from paper_2504_06095_b200.linear import partner_row_map
    fused = []
    for li in range(L):
        per = []
        for (sh, X, G, grads), s in zip(shards[li], groups[li].hosted):
            healthy = s < n1
            cols = hc[s] if healthy else rc[s - n1]
            partner_cols = rc if healthy else hc
            partner_slots = [n1 + j for j in range(n2)] if healthy else list(range(n1))
            ptrs = groups[li].open_slots(partner_slots)
            sptrs = staging[li].open_slots(partner_slots)
            rb, rr = partner_row_map(cols, partner_cols, "cuda")
            per.append((sh, X, G, grads, w_h if healthy else w_r, rb, rr, ptrs, sptrs,
                        staging[li].arena(s)))
        fused.append(per)

    class _P:  # raw pointer holder with the .data_ptr() mm_red expects
        def __init__(self, p):
            self.p = p

        def data_ptr(self):
            return self.p

    from paper_2504_06095_b200.linear import finish_push

    def fused_backward(mode="red"):
        for li in range(L):
            gr = groups[li]
            gr.epoch += 1
            if mode == "red":
                for s in gr.hosted:
                    gr.arena(s).zero_()
            gr.signal("post_ready", gr.epoch, main)
            gr.signal("wait_ready", gr.epoch, main)
        for li in reversed(range(L)):
            for sh, X, G, grads, alpha, rb, rr, ptrs, sptrs, st in fused[li]:
                tgt = ptrs if mode == "red" else sptrs
                sh.backward_synced(X, G, grads, alpha, rb, rr, [_P(p) for p in tgt], main, mode)
            groups[li].signal("post_done", groups[li].epoch, main)
        for li in range(L):
            groups[li].signal("wait_done", groups[li].epoch, main)
            if mode == "push":
                for sh, X, G, grads, alpha, rb, rr, ptrs, sptrs, st in fused[li]:
                    finish_push(grads, st, main)

    def timed(fn, iters):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for _ in range(iters):
            fn()
        e1.record(main)
        torch.cuda.synchronize()
        ms = tmax(e0.elapsed_time(e1) / iters)
        dist.barrier()
        return ms

    Lb = _lib.load()
    res = {"n1": n1, "n2": n2, "tokens_healthy": tok_h, "tokens_degraded": tok_r,
           "placement_healthy": list(plc.h_proc), "placement_reduced": list(plc.r_proc)}
    res["backward_ms"] = round(timed(lambda: backward(False, sync=False), args.iters), 3)
    res["sync_ms"] = round(timed(sync_only, args.iters), 3)
    res["serial_ms"] = round(timed(lambda: backward(False), args.iters), 3)
    res["fused_wgrad_sync_ms"] = round(timed(fused_backward, args.iters), 3)
    res["fused_push_wgrad_sync_ms"] = round(timed(lambda: fused_backward("push"), args.iters), 3)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    for cap in args.caps:
        # TMA-bulk sync (131 KB smem/CTA): it cannot share an SM with a GEMM CTA,
        # so the sync gets `cap` SMs and the persistent GEMMs the remaining ones
        Lb.ntp_set_option(0, 2)
        Lb.ntp_set_option(1, cap)
        Lb.ntp_gemm_set_max_ctas(sms - cap if cap else 0)
        res[f"overlap_ms_bulk_cap{cap}"] = round(timed(lambda: backward(True), args.iters), 3)
    Lb.ntp_gemm_set_max_ctas(0)
    for cap in args.ldg_caps:
        # register-staged sync (no smem): its CTAs co-reside with the GEMM's
        # 1 CTA/SM, so the GEMMs keep every SM
        Lb.ntp_set_option(0, 1)
        Lb.ntp_set_option(1, cap)
        res[f"overlap_ms_ldg_cap{cap}"] = round(timed(lambda: backward(True), args.iters), 3)
    Lb.ntp_set_option(0, 1)
    Lb.ntp_set_option(1, 74)
    for _ in range(2):
        timeline()
    tl = timeline()
    allt = [None] * dist.get_world_size()
    dist.all_gather_object(allt, tl)
    res["timeline_ldg_cap74_per_rank"] = allt
    Lb.ntp_set_option(0, 0)
    Lb.ntp_set_option(1, 0)
    for gr in groups + staging:
        assert gr.status() == 0, "signal timeout"
        gr.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--caps", type=int, nargs="*", default=[16])
    ap.add_argument("--ldg-caps", type=int, nargs="*", default=[32, 74, 148, 296])
    args = ap.parse_args()
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = dist.get_world_size()
    n1 = max(1, world // 2)
    ntp = run_config(args, n1, n1 - 1, local) if n1 > 1 else None
    uni = run_config(args, n1, n1, local)
    if dist.get_rank() == 0:
        best = lambda r: min(v for key, v in r.items()  # noqa: E731
                             if key.startswith("overlap_ms") or key.startswith("fused"))
        doc = {"world": world, "layers": args.layers, "hidden": args.hidden, "ffn": args.ffn,
               "ntp": ntp, "uniform": uni}
        if ntp:
            doc["step_overhead_ntp_vs_uniform"] = round(best(ntp) / best(uni) - 1.0, 4)
            doc["exposed_sync_ms_ntp"] = round(best(ntp) - ntp["backward_ms"], 3)
            doc["exposed_sync_ms_uniform"] = round(best(uni) - uni["backward_ms"], 3)
        print(json.dumps(doc, indent=1), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
