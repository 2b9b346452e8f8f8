"""Split-K tail sweep: each C4 GEMM timed with split off and capped at 2/4/8
pieces (ntp_gemm_set_split_k).  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib, linear as L  # noqa: E402
from gemm_bench import timed  # noqa: E402


def main():
    T, h = 8192, 4096
    g = torch.Generator(device="cuda").manual_seed(0)
    out = []
    lib = _lib.load()
    for n in (4779, 3584):
        npad = (n + 7) // 8 * 8
        X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
        G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
        W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
        Hb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
        Yb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
        Z = torch.empty((T, h), dtype=torch.float32, device="cuda")
        grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
        cases = [("fwd1", lambda: L.mm(X, W[:, 0, :], Yb, epilogue="gelu", aux=Hb), T, n, h),
                 ("fwd2", lambda: L.mm(Yb, W[:, 1, :].T, Z), T, h, n),
                 ("wgrad", lambda: L.mm(Yb.T, G.T, grads[:, 1, :]), n, h, T)]
        for name, fn, M, N, K in cases:
            r = {"n_i": n, "gemm": name, "M": M, "N": N, "K": K}
            for cap in (0, 2, 4, 8):
                lib.ntp_gemm_set_split_k(cap)
                ms = timed(fn)
                r[f"split{cap}_tflops"] = round(2.0 * M * N * K / ms / 1e9, 1)
            lib.ntp_gemm_set_split_k(1)
            out.append(r)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
