"""Degraded-replica step overhead (north_star: <= 5 % over uniform TP).

One process per GPU (torchrun).  Two DP replicas of an L-layer MLP stack
(hidden h, ffn k; the reference's 2-matrix GeLU MLP, tpnumerics.py:177-252):

  * NTP:      healthy TP-n1 + degraded TP-n2 (local batch scaled by n2/n1,
              so every GPU does the same GEMM work; policy.py:139-148 shrinks
              the reduced replica's batch the same way)
  * uniform:  healthy TP-n1 + healthy TP-n1

Per layer, in reverse order, every GPU runs its shard's backward on the tensor
cores (D = (G B^T) * GeLU'(H); dB = Y^T G and dA^T = D^T X written straight
into the layer's unit-major gradient arena) and that layer's gradient sync.
Modes (device time per step, max over ranks):

  backward        GEMMs only (no sync) -- the floor
  sync_only       the 8 layer syncs alone (dist.NtpSyncGroup)
  serial          GEMMs, then the syncs
  overlap_*       each layer's sync on a high-priority side stream under the
                  next layers' GEMMs (bulk kernel on capped SMs, or the
                  register-staged kernel co-resident with the GEMM CTAs)
  fused_red       wgrad epilogue red.adds into both replicas' zeroed arenas
  fused_push      wgrad epilogue row-stores into the partner's staging arena,
                  the layer's local tail (arena += staging) on the side stream
  fused_push_tma  the same with 32-row boxes sent as TMA tensor stores over NVLink

The two configurations are built side by side and every mode is timed NTP then
uniform back to back, for several rounds; the minimum per mode is kept, so
slow drifts (clocks, power) hit both sides alike.  overhead = best NTP mode /
best uniform mode - 1, and per mode.

    torchrun --nproc-per-node 4 scripts/step_bench.py [--layers 8 --tokens 8192 --rounds 3]
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
from paper_2504_06095_b200.linear import MlpShard, finish_push, partner_row_map  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class _P:  # raw pointer holder with the .data_ptr() mm_red expects
    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


class Config:
    """One DP=2 configuration (TP-n1 + TP-n2) of the L-layer MLP stack."""

    def __init__(self, args, n1, n2, local, main, side):
        rank = dist.get_rank()
        h, k, L = args.hidden, args.ffn, args.layers
        self.n1, self.n2, self.L, self.main, self.side = n1, n2, L, main, side
        shape = ModelShape("step", h, k, 0, 1)
        lay = pair_layout(shape, n1, n2)
        self.plc = plc = Placement.default(dist.get_world_size(), n1, n2)
        self.tok_h = tok_h = args.tokens
        self.tok_r = tok_r = args.tokens * n2 // n1
        self.w_h, self.w_r = tok_h / (tok_h + tok_r), tok_r / (tok_h + tok_r)
        self.groups = [NtpSyncGroup(lay, plc, torch.bfloat16, local).upload() for _ in range(L)]
        self.staging = [NtpSyncGroup(lay, plc, torch.bfloat16, local).upload() for _ in range(L)]
        g = torch.Generator(device="cuda").manual_seed(rank)
        rng = np.random.default_rng(rank)
        Xh = torch.randn((tok_h, h), generator=g, device="cuda").to(torch.bfloat16)
        Gh = torch.randn((tok_h, h), generator=g, device="cuda").to(torch.bfloat16)
        Xr = torch.randn((tok_r, h), generator=g, device="cuda").to(torch.bfloat16)
        Gr = torch.randn((tok_r, h), generator=g, device="cuda").to(torch.bfloat16)
        A = rng.standard_normal((h, k)) / np.sqrt(h)
        B = rng.standard_normal((k, h)) / np.sqrt(k)
        _k, _unit, hc, rc, _hb, _rb = lay.segs[0]
        self.shards, self.fused = [], []
        for li in range(L):
            per, fper = [], []
            for s in self.groups[li].hosted:
                healthy = s < n1
                cols = hc[s] if healthy else rc[s - n1]
                sh = MlpShard(A, B, cols)
                X, G = (Xh, Gh) if healthy else (Xr, Gr)
                Z = torch.empty((X.shape[0], h), dtype=torch.float32, device="cuda")
                sh.forward(X, Z)  # H, Y for the backward
                grads = self.groups[li].arena(s).view(len(cols), 2, h)
                per.append((sh, X, G, grads))
                partner_cols = rc if healthy else hc
                partner_slots = [n1 + j for j in range(n2)] if healthy else list(range(n1))
                ptrs = self.groups[li].open_slots(partner_slots)
                sptrs = self.staging[li].open_slots(partner_slots)
                rb, rr = partner_row_map(cols, partner_cols, "cuda")
                fper.append((sh, X, G, grads, self.w_h if healthy else self.w_r, rb, rr, ptrs,
                             sptrs, self.staging[li].arena(s)))
            self.shards.append(per)
            self.fused.append(fper)

    def backward(self, overlap: bool, sync: bool = True, pdl: bool = False):
        main, side = self.main, self.side
        for li in reversed(range(self.L)):
            for sh, X, G, grads in self.shards[li]:
                # PDL chain: each layer's first GEMM shares no data with the
                # previous layer's last one (G is given, D is per shard)
                sh.backward(X, G, grads, pdl="independent" if pdl else None)
            if sync and overlap:
                side.wait_stream(main)
                self.groups[li].step(self.w_h, self.w_r, side)
        if sync and not overlap:
            for li in reversed(range(self.L)):
                self.groups[li].step(self.w_h, self.w_r, main)
        main.wait_stream(side)

    def sync_only(self):
        for li in reversed(range(self.L)):
            self.groups[li].step(self.w_h, self.w_r, self.main)

    def fused_backward(self, mode="red"):
        main, side = self.main, self.side
        red = mode in ("red", "red_tma")
        if red:
            # zero each layer's arena on the side stream (in backward order) and
            # tell the partners; a layer's GEMMs wait for both ends' zeroing
            side.wait_stream(main)
            zeroed = {}
            for li in reversed(range(self.L)):
                gr = self.groups[li]
                gr.epoch += 1
                with torch.cuda.stream(side):
                    for s in gr.hosted:
                        gr.arena(s).zero_()
                gr.signal("post_ready", gr.epoch, side)
                ev = torch.cuda.Event()
                ev.record(side)
                zeroed[li] = ev
        else:
            for li in range(self.L):
                gr = self.groups[li]
                gr.epoch += 1
                gr.signal("post_ready", gr.epoch, main)
                gr.signal("wait_ready", gr.epoch, main)
        for li in reversed(range(self.L)):
            if red:
                main.wait_event(zeroed[li])
                self.groups[li].signal("wait_ready", self.groups[li].epoch, main)
            for sh, X, G, grads, alpha, rb, rr, ptrs, sptrs, st in self.fused[li]:
                tgt = ptrs if mode in ("red", "red_tma") else sptrs
                sh.backward_synced(X, G, grads, alpha, rb, rr, [_P(p) for p in tgt], main, mode)
            self.groups[li].signal("post_done", self.groups[li].epoch, main)
            if mode in ("push", "push_tma"):
                # the layer's local tail (arena += partner's staging) runs on the
                # side stream under the next layers' GEMMs
                side.wait_stream(main)
                self.groups[li].signal("wait_done", self.groups[li].epoch, side)
                for sh, X, G, grads, alpha, rb, rr, ptrs, sptrs, st in self.fused[li]:
                    finish_push(grads, st, side)
        if mode in ("red", "red_tma"):
            for li in range(self.L):
                self.groups[li].signal("wait_done", self.groups[li].epoch, main)
        else:
            main.wait_stream(side)

    def timeline(self):
        """One overlapped backward with events: per layer, when its GEMMs and its
        sync finished (ms from the start), on this rank."""
        main, side = self.main, self.side
        t0 = torch.cuda.Event(enable_timing=True)
        g_end, s_end = [], []
        torch.cuda.synchronize()
        dist.barrier()
        t0.record(main)
        for li in reversed(range(self.L)):
            for sh, X, G, grads in self.shards[li]:
                sh.backward(X, G, grads)
            e = torch.cuda.Event(enable_timing=True)
            e.record(main)
            g_end.append(e)
            side.wait_event(e)
            self.groups[li].step(self.w_h, self.w_r, side)
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record(side)
            s_end.append(e2)
        main.wait_stream(side)
        torch.cuda.synchronize()
        return {"gemm_done_ms": [round(t0.elapsed_time(e), 3) for e in g_end],
                "sync_done_ms": [round(t0.elapsed_time(e), 3) for e in s_end]}

    def product(self, uncap_last=True, sync_ctas=16):
        """The package's OverlappedBackward over this configuration."""
        if getattr(self, "_ob", None) is None:
            from paper_2504_06095_b200.step import OverlappedBackward
            layers = [(self.groups[li], [(sh, grads) for sh, X, G, grads in self.shards[li]])
                      for li in range(self.L)]
            self._ob = OverlappedBackward(layers, self.w_h, self.w_r)
            self._ob_inputs = [[(X, G) for sh, X, G, grads in self.shards[li]]
                               for li in range(self.L)]
        self._ob.uncap_last = uncap_last
        self._ob.sync_ctas = sync_ctas
        self._ob.run(self._ob_inputs, self.main)

    def set_policy(self, policy):
        if self.groups[0].policy != policy:
            for gr in self.groups:
                gr.set_policy(policy)

    def describe(self):
        return {"n1": self.n1, "n2": self.n2, "tokens_healthy": self.tok_h,
                "tokens_degraded": self.tok_r, "placement_healthy": list(self.plc.h_proc),
                "placement_reduced": list(self.plc.r_proc)}

    def close(self):
        for gr in self.groups + self.staging:
            assert gr.status() == 0, "signal timeout"
            gr.close()


def timed(main, fn, iters):
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


def modes(Lb, sms):
    """name -> (setup(), run(cfg)[, executor policy]).  setup sets the global
    kernel options; the policy (default "split") is applied to both configs."""
    def opts(kernel=0, cap=0, gemm_cap=0):
        def f():
            Lb.ntp_set_option(0, kernel)
            Lb.ntp_set_option(1, cap)
            Lb.ntp_gemm_set_max_ctas(gemm_cap)
        return f
    return {
        "backward": (opts(), lambda c: c.backward(False, sync=False)),
        "backward_pdl": (opts(), lambda c: c.backward(False, sync=False, pdl=True)),
        "sync_only": (opts(), lambda c: c.sync_only()),
        "serial": (opts(), lambda c: c.backward(False)),
        # TMA-bulk sync (131 KB smem/CTA) cannot share an SM with a GEMM CTA:
        # it gets 16 SMs and the persistent GEMMs the rest
        "overlap_bulk_cap16": (opts(2, 16, sms - 16), lambda c: c.backward(True)),
        # register-staged sync (no smem) co-resides with the GEMM's 1 CTA/SM
        "overlap_ldg_cap148": (opts(1, 148), lambda c: c.backward(True)),
        "overlap_ldg_cap296": (opts(1, 296), lambda c: c.backward(True)),
        # executor policy "healthy": the degraded GPU computes no sync units
        "overlap_bulk_cap16_healthy": (opts(2, 16, sms - 16), lambda c: c.backward(True),
                                       "healthy"),
        "overlap_ldg_cap148_healthy": (opts(1, 148), lambda c: c.backward(True), "healthy"),
        # the same configuration through the package API (step.OverlappedBackward)
        "product_overlapped": (opts(), lambda c: c.product(), "healthy"),
        "product_overlapped_capped_last": (opts(), lambda c: c.product(False), "healthy"),
        "product_overlapped_sync8": (opts(), lambda c: c.product(True, 8), "healthy"),
        "product_overlapped_sync24": (opts(), lambda c: c.product(True, 24), "healthy"),
        "product_overlapped_sync32": (opts(), lambda c: c.product(True, 32), "healthy"),
        "overlap_bulk_cap16_healthy_pdl": (opts(2, 16, sms - 16),
                                           lambda c: c.backward(True, pdl=True), "healthy"),
        "fused_red": (opts(), lambda c: c.fused_backward("red")),
        "fused_push": (opts(), lambda c: c.fused_backward("push")),
        "fused_push_tma": (opts(), lambda c: c.fused_backward("push_tma")),
        "fused_red_tma": (opts(), lambda c: c.fused_backward("red_tma")),
        "fused_push_tma_ldg_cap74": (opts(1, 74), lambda c: c.fused_backward("push_tma")),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = dist.get_world_size()
    n1 = max(1, world // 2)
    if n1 < 2:
        raise SystemExit("needs >= 4 GPUs (TP2 + TP1 vs TP2 + TP2)")
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=-1)  # sync CTAs are scheduled ahead of GEMM CTAs
    ntp = Config(args, n1, n1 - 1, local, main_s, side)
    uni = Config(args, n1, n1, local, main_s, side)
    torch.cuda.synchronize()
    dist.barrier()
    Lb = _lib.load()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    table = modes(Lb, sms)
    best = {name: [float("inf"), float("inf")] for name in table}
    from bench import ClockSampler  # repo root is on sys.path
    clocks = ClockSampler(local)
    clocks.start()
    clocks.mark("t0")
    for _ in range(args.rounds):
        for name, (setup, run, *pol) in table.items():
            setup()
            for j, cfg in enumerate((ntp, uni)):
                cfg.set_policy(pol[0] if pol else "split")
                best[name][j] = min(best[name][j], timed(main_s, lambda: run(cfg), args.iters))
    for cfg in (ntp, uni):
        cfg.set_policy("split")
    clocks.mark("t1")
    clk = clocks.stop()
    all_clk = [None] * world
    dist.all_gather_object(all_clk, clk)
    Lb.ntp_set_option(0, 1)
    Lb.ntp_set_option(1, 148)
    Lb.ntp_gemm_set_max_ctas(0)
    tls = []
    for cfg in (ntp, uni):
        for _ in range(2):
            cfg.timeline()
        tl = cfg.timeline()
        allt = [None] * world
        dist.all_gather_object(allt, tl)
        tls.append(allt)
    Lb.ntp_set_option(0, 0)
    Lb.ntp_set_option(1, 0)
    if dist.get_rank() == 0:
        step_modes = [m for m in table if m.startswith(("overlap", "fused"))]
        res = {"world": world, "layers": args.layers, "hidden": args.hidden, "ffn": args.ffn,
               "tokens": args.tokens, "rounds": args.rounds, "iters": args.iters,
               "ntp": ntp.describe(), "uniform": uni.describe(),
               "ms": {m: {"ntp": round(v[0], 3), "uniform": round(v[1], 3),
                          "overhead": round(v[0] / v[1] - 1.0, 4)} for m, v in best.items()}}
        bn = min(step_modes, key=lambda m: best[m][0])
        bu = min(step_modes, key=lambda m: best[m][1])
        res["best_ntp"] = {"mode": bn, "ms": round(best[bn][0], 3)}
        res["best_uniform"] = {"mode": bu, "ms": round(best[bu][1], 3)}
        res["step_overhead_ntp_vs_uniform"] = round(best[bn][0] / best[bu][1] - 1.0, 4)
        res["exposed_sync_ms_ntp"] = round(best[bn][0] - best["backward"][0], 3)
        res["exposed_sync_ms_uniform"] = round(best[bu][1] - best["backward"][1], 3)
        res["clocks_per_rank"] = all_clk
        res["timeline_ldg_cap148_per_rank"] = {"ntp": tls[0], "uniform": tls[1]}
        print(json.dumps(res, indent=1), flush=True)
    dist.barrier()
    ntp.close()
    uni.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
