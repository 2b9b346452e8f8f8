"""tcgen05 GEMM throughput on the C4 (Llama-3-8B-shaped) per-rank MLP GEMMs,
next to cuBLAS (torch.matmul) on the same shapes.  Prints JSON.

    python scripts/gemm_bench.py [tokens]
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import linear as L  # noqa: E402

PEAK = 1661.5  # MEASURED_PEAKS.json bf16 burst
PEAK_SUSTAINED = 1388.7  # MEASURED_PEAKS.json: cuBLAS 8192^3 back to back for 4 s (power-capped)


def timed(fn, iters=20):
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


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    h = 4096
    import bench
    clocks = bench.ClockSampler(0)
    clocks.start()
    clocks.mark("t0")
    out = {"tokens": T, "hidden": h, "peak_tflops": PEAK, "peak_tflops_sustained": PEAK_SUSTAINED,
           "gemms": []}
    g = torch.Generator(device="cuda").manual_seed(0)
    for n in (4779, 3584):
        npad = (n + 7) // 8 * 8
        X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
        G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
        W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
        Hb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
        Yb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
        Db = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
        Z = torch.empty((T, h), dtype=torch.float32, device="cuda")
        grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
        cases = [
            ("fwd1 H=X A_i (+GeLU)", lambda: L.mm(X, W[:, 0, :], Yb, epilogue="gelu", aux=Hb),
             lambda: torch.matmul(X, W[:, 0, :].T), T, n, h),
            ("fwd2 Z=Y B_i (fp32 out)", lambda: L.mm(Yb, W[:, 1, :].T, Z),
             lambda: torch.matmul(Yb, W[:, 1, :]), T, h, n),
            ("bwd D=(G B_i^T)*GeLU'(H)", lambda: L.mm(G, W[:, 1, :], Db, epilogue="dgelu", aux=Hb),
             lambda: torch.matmul(G, W[:, 1, :].T), T, n, h),
            ("wgrad dB_i=Y^T G (unit-major)", lambda: L.mm(Yb.T, G.T, grads[:, 1, :]),
             lambda: torch.matmul(Yb.T, G), n, h, T),
            ("wgrad dA_i=D^T X (unit-major)", lambda: L.mm(Db.T, X.T, grads[:, 0, :]),
             lambda: torch.matmul(Db.T, X), n, h, T),
        ]
        from paper_2504_06095_b200 import _lib
        for name, ours, ref, M, N, K in cases:
            fl = 2.0 * M * N * K
            modes = {}
            for mode, name_m in ((0, "single_256"), (2, "pair_128"), (3, "pair_256"), (4, "pair_224"),
                                 (1, "auto")):
                _lib.load().ntp_gemm_set_pair(mode)
                modes[name_m] = timed(ours)
            _lib.load().ntp_gemm_set_split_k(0)
            modes["auto_nosplit"] = timed(ours)
            _lib.load().ntp_gemm_set_split_k(1)
            ms1 = modes["single_256"]
            ms = modes["auto"]
            ms_ref = timed(ref)

            out["gemms"].append({"n_i": n, "gemm": name, "M": M, "N": N, "K": K,
                                 "ours_ms": round(ms, 4), "ours_tflops": round(fl / ms / 1e9, 1),
                                 "ours_frac": round(fl / ms / 1e9 / PEAK, 3),
                                 "ours_frac_sustained": round(fl / ms / 1e9 / PEAK_SUSTAINED, 3),
                                 "single_cta_tflops": round(fl / ms1 / 1e9, 1),
                                 "tflops_by_tile": {k: round(fl / v / 1e9, 1)
                                                    for k, v in modes.items()},
                                 "cublas_ms": round(ms_ref, 4),
                                 "cublas_tflops": round(fl / ms_ref / 1e9, 1)})
    clocks.mark("t1")
    out["clocks"] = clocks.stop()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
