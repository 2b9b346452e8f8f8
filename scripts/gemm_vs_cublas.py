"""tcgen05 GEMM vs cuBLAS on the C4 per-rank MLP GEMMs, interleaved, with the
SM clock sampled (NVML) during every measurement, so a throughput gap can be
told apart from a clock (power-cap) gap.  cuBLAS gets contiguous operands padded
to a multiple of 8 columns (its fast kernels need 16-byte aligned rows); ours
runs on the strided unit-major views the NTP path uses.  Prints JSON.

    python scripts/gemm_vs_cublas.py [rounds] [raster,...] [epi_sleep,...]
"""

import ctypes
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200 import linear as L  # noqa: E402


class Clock:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

    def sample(self, fn, iters):
        vals, stop = [], [False]

        def loop():
            while not stop[0]:
                vals.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                time.sleep(0.002)
        th = threading.Thread(target=loop, daemon=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        th.start()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        stop[0] = True
        th.join()
        vals.sort()
        return e0.elapsed_time(e1) / iters, (vals[len(vals) // 2] if vals else None)


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    rasters = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
    sleeps = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1]
    variants = [(r, s) for r in rasters for s in sleeps]
    lib = _lib.load()
    lib.ntp_gemm_debug_raster.argtypes = [ctypes.c_int]
    lib.ntp_gemm_debug_epi_sleep.argtypes = [ctypes.c_int]
    T, h = 8192, 4096
    clock = Clock()
    g = torch.Generator(device="cuda").manual_seed(0)
    out = {"tokens": T, "hidden": h, "rounds": rounds, "gemms": []}
    for n in (4779, 3584):
        npad = (n + 7) // 8 * 8
        X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
        G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
        W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
        Hb = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)[:, :n]
        Yb = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)[:, :n]
        Db = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
        Z = torch.empty((T, h), dtype=torch.float32, device="cuda")
        grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
        # cuBLAS operands: contiguous, padded to npad
        Wa = torch.randn((npad, h), generator=g, device="cuda").to(torch.bfloat16)
        Wb = torch.randn((npad, h), generator=g, device="cuda").to(torch.bfloat16)
        Yc = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)
        cases = [
            ("fwd1", lambda: L.mm(X, W[:, 0, :], Yb, epilogue="gelu", aux=Hb),
             lambda: torch.matmul(X, Wa.T), T, n, h),
            ("fwd2", lambda: L.mm(Yb, W[:, 1, :].T, Z),
             lambda: torch.matmul(Yc, Wb), T, h, n),
            ("bwd_dgelu", lambda: L.mm(G, W[:, 1, :], Db, epilogue="dgelu", aux=Hb),
             lambda: torch.matmul(G, Wb.T), T, n, h),
            ("wgrad_dB", lambda: L.mm(Yb.T, G.T, grads[:, 1, :]),
             lambda: torch.matmul(Yc.T, G), n, h, T),
            ("wgrad_dA", lambda: L.mm(Db.T, X.T, grads[:, 0, :]),
             lambda: torch.matmul(Yc.T, X), n, h, T),
        ]
        for name, ours, ref, M, N, K in cases:
            fl = 2.0 * M * N * K
            iters = max(10, int(40e-3 / (fl / 1.3e15)))  # ~40 ms per measurement
            rec = {"n_i": n, "gemm": name, "M": M, "N": N, "K": K, "iters": iters}
            for _ in range(3):
                ours()
                ref()
            best = {}
            for _ in range(rounds):
                for r, sl in variants:
                    lib.ntp_gemm_debug_raster(r)
                    lib.ntp_gemm_debug_epi_sleep(sl)
                    ms, mhz = clock.sample(ours, iters)
                    key = f"ours_r{r}s{sl}"
                    if key not in best or ms < best[key][0]:
                        best[key] = (ms, mhz)
                ms, mhz = clock.sample(ref, iters)
                if "cublas" not in best or ms < best["cublas"][0]:
                    best["cublas"] = (ms, mhz)
            lib.ntp_gemm_debug_raster(0)
            lib.ntp_gemm_debug_epi_sleep(1)
            for k, (ms, mhz) in best.items():
                fl_k = fl if k != "cublas" else 2.0 * (M if M != n else npad) * (N if N != n else npad) * (K if K != n else npad)
                tf = fl_k / ms / 1e9
                rec[k] = {"ms": round(ms, 4), "tflops": round(tf, 1), "sm_mhz": mhz,
                          "tflops_per_ghz": round(tf / (mhz / 1e3), 1) if mhz else None}
            out["gemms"].append(rec)
            print(json.dumps(rec), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
