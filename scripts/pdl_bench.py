"""Backward GEMM chain with and without programmatic dependent launch, one GPU,
interleaved A/B rounds (same clocks for both).  8 layers x 3 GEMMs of a TP2
shard of the C4 MLP (n = 7168 of ffn 14336, h = 4096, 8192 tokens).  JSON out."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06095_b200 import linear as L  # noqa: E402


def main():
    layers, T, h, n = 8, 8192, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 7168
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
    G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
    shards, grads = [], []
    rng = np.random.default_rng(0)
    A = rng.standard_normal((h, n)).astype(np.float32) / 64
    B = rng.standard_normal((n, h)).astype(np.float32) / 64
    for _ in range(layers):
        sh = L.MlpShard(A, B, np.arange(n))
        sh.forward(X, torch.empty((T, h), dtype=torch.float32, device="cuda"))
        shards.append(sh)
        grads.append(torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda"))

    def chain(pdl):
        for li in reversed(range(layers)):
            shards[li].backward(X, G, grads[li], pdl="independent" if pdl else None)

    def timed(pdl, iters=5):
        chain(pdl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            chain(pdl)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    res = {"off": [], "pdl": []}
    for _ in range(6):
        res["off"].append(timed(False))
        res["pdl"].append(timed(True))
    fl = layers * 3 * 2.0 * T * n * h
    out = {"layers": layers, "tokens": T, "hidden": h, "n_shard": n,
           "ms_off": [round(x, 3) for x in res["off"]], "ms_pdl": [round(x, 3) for x in res["pdl"]],
           "min_off": round(min(res["off"]), 3), "min_pdl": round(min(res["pdl"]), 3),
           "median_off": round(float(np.median(res["off"])), 3),
           "median_pdl": round(float(np.median(res["pdl"])), 3),
           "tflops_off": round(fl / min(res["off"]) / 1e9, 1),
           "tflops_pdl": round(fl / min(res["pdl"]) / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
