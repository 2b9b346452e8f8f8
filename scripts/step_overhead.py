"""Degraded-replica step overhead against a uniform-TP NCCL comparator
(north_star: <= 5 %; PAPER.md:382 reports <= 4 % final-backward slowdown).

One process per GPU (torchrun).  Two DP replicas of an L-layer stack whose
layers carry an MLP partition (k = ffn columns, 2h-element units) and an
attention partition (k = heads, 4*h*hd-element units), bf16:

  * NTP       healthy TP-n1 + degraded TP-n2 (local batch x n2/n1, so every
              GPU does the same GEMM work), each layer's sync = the NVLink
              peer-memory nonuniform sync (dist.NtpSyncGroup, policy "healthy")
  * uniform   healthy TP-n1 + healthy TP-n1, each layer's sync = NCCL
              all-reduce of the aligned shards (NtpSyncGroup(aligned="nccl"):
              what a uniform deployment runs)

Both run the package's overlapped backward (step.OverlappedBackward): per
layer, in reverse order, the tcgen05 backward GEMMs of the MLP shard write
the unit-major arena, and the layer's sync runs on a high-priority side stream
under the next layers' GEMMs.  Attention-head units are synced (their bytes
are in every layer's arena) but have no GEMM here (attention backward is not
on this path).  Rounds interleave the configurations; each round times
`--steps` whole backward steps per configuration (device time, max over
ranks).  Reported: per-round overhead NTP / uniform - 1, its median and IQR,
and the SM clocks each rank saw.

    torchrun --nproc-per-node 4 scripts/step_overhead.py [--n1 4 --n2 3 --rounds 10]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2504_06095_b200.dist import NtpSyncGroup, Placement  # noqa: E402
from paper_2504_06095_b200.linear import MlpShard  # noqa: E402
from paper_2504_06095_b200.step import OverlappedBackward  # noqa: E402
from paper_2504_06095_b200.workloads import ModelShape, pair_layout  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class Config:
    def __init__(self, args, n1, n2, aligned, local):
        rank = dist.get_rank()
        h, k, L = args.hidden, args.ffn, args.layers
        shape = ModelShape("step", h, k, args.heads, 1)
        lay = pair_layout(shape, n1, n2)
        plc = Placement.default(dist.get_world_size(), n1, n2)
        self.describe = {"n1": n1, "n2": n2, "sync": "nccl all-reduce" if aligned == "nccl"
                         else "peer-memory nonuniform sync", "placement_healthy": list(plc.h_proc),
                         "placement_reduced": list(plc.r_proc)}
        tok_h, tok_r = args.tokens, args.tokens * n2 // n1
        self.w_h, self.w_r = tok_h / (tok_h + tok_r), tok_r / (tok_h + tok_r)
        self.describe.update(tokens_healthy=tok_h, tokens_degraded=tok_r)
        # uniform NCCL: the batch weight rides on the wgrad GEMMs' alpha and the
        # all-reduce is a plain SUM (prescaled), as a uniform deployment would do
        self.groups = [NtpSyncGroup(lay, plc, torch.bfloat16, local, aligned=aligned,
                                    prescaled=aligned == "nccl").upload() for _ in range(L)]
        g = torch.Generator(device="cuda").manual_seed(rank)
        rng = np.random.default_rng(rank)
        X = {s: torch.randn((tok_h if s < n1 else tok_r, h), generator=g, device="cuda")
             .to(torch.bfloat16) for s in range(n1 + n2)}
        G = {s: torch.randn((tok_h if s < n1 else tok_r, h), generator=g, device="cuda")
             .to(torch.bfloat16) for s in range(n1 + n2)}
        A = rng.standard_normal((h, k)) / np.sqrt(h)
        B = rng.standard_normal((k, h)) / np.sqrt(k)
        _k, _unit, hc, rc, _hb, _rb = lay.segs[0]
        layers, inputs = [], []
        for li in range(L):
            per, inp = [], []
            gr = self.groups[li]
            for s in gr.hosted:
                a = gr.arena(s)
                a.copy_(torch.randn(a.numel(), generator=g, device="cuda").to(torch.bfloat16))
                cols = hc[s] if s < n1 else rc[s - n1]
                sh = MlpShard(A, B, cols)
                sh.activations(X[s])
                grads = a[:len(cols) * 2 * h].view(len(cols), 2, h)  # the MLP segment
                per.append((sh, grads))
                inp.append((X[s], G[s]))
            layers.append((gr, per))
            inputs.append(inp)
        self.inputs = inputs
        self.ob = OverlappedBackward(layers, self.w_h, self.w_r)
        self.floor_layers = layers

    def step(self, main):
        self.ob.run(self.inputs, main)

    def gemms_only(self, main):
        with torch.cuda.stream(main):
            for li in reversed(range(len(self.floor_layers))):
                for (sh, grads), (X, G) in zip(self.floor_layers[li][1], self.inputs[li]):
                    sh.backward(X, G, grads)

    def close(self):
        for gr in self.groups:
            assert gr.status() == 0, "signal timeout"
            gr.close()


def timed(main, fn, steps):
    for _ in range(2):
        fn(main)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(steps):
        fn(main)
    e1.record(main)
    torch.cuda.synchronize()
    return tmax(e0.elapsed_time(e1) / steps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--n1", type=int, default=4)
    ap.add_argument("--n2", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    os.environ["NCCL_DEBUG"] = "WARN"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    main_s = torch.cuda.current_stream()
    cfgs = {"ntp": Config(args, args.n1, args.n2, "peer", local),
            "uniform_nccl": Config(args, args.n1, args.n1, "nccl", local),
            "uniform_peer": Config(args, args.n1, args.n1, "peer", local)}
    clocks = ClockSampler(local)
    clocks.start()
    clocks.mark("t0")
    res = {f"{n}_{m}": [] for n in cfgs for m in ("step", "gemms")}
    for _ in range(args.rounds):
        for name, c in cfgs.items():
            res[f"{name}_step"].append(timed(main_s, c.step, args.steps))
            res[f"{name}_gemms"].append(timed(main_s, c.gemms_only, args.steps))
    clocks.mark("t1")
    clk = clocks.stop()
    clk_all = [None] * dist.get_world_size()
    dist.all_gather_object(clk_all, clk)
    ov = np.array(res["ntp_step"]) / np.array(res["uniform_nccl_step"]) - 1
    ovp = np.array(res["ntp_step"]) / np.array(res["uniform_peer_step"]) - 1
    if rank == 0:
        q = lambda a: [round(float(np.percentile(a, p)), 4) for p in (25, 50, 75)]  # noqa: E731
        out = {"what": "degraded-replica overlapped backward step vs uniform TP (NCCL all-reduce "
                       "comparator), interleaved rounds, device ms per step, max over ranks",
               "n_gpus": dist.get_world_size(), "layers": args.layers, "tokens": args.tokens,
               "hidden": args.hidden, "ffn": args.ffn, "heads": args.heads,
               "configs": {n: c.describe for n, c in cfgs.items()},
               "ms": {k: [round(x, 4) for x in v] for k, v in res.items()},
               "median_ms": {k: round(float(np.median(v)), 4) for k, v in res.items()},
               "overhead_vs_uniform_nccl": {"per_round": [round(float(x), 4) for x in ov],
                                            "q25_median_q75": q(ov)},
               "overhead_vs_uniform_peer": {"per_round": [round(float(x), 4) for x in ovp],
                                            "q25_median_q75": q(ovp)},
               "clocks_per_rank": clk_all}
        print(json.dumps(out, indent=1), flush=True)
    for c in cfgs.values():
        c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
