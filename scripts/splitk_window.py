"""fwd1-shaped GEMM (8192 x 4779 x 4096, GeLU epilogue): split-K cap x fixup
wait window (debug hook ntp_gemm_debug_split_window), interleaved rounds."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib, linear as L  # noqa: E402
from gemm_bench import timed  # noqa: E402

lib = _lib.load()
fn = lib.ntp_gemm_debug_split_window
fn.argtypes = [ctypes.c_ulonglong]
T, h, n = 8192, 4096, 4779
npad = (n + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
Hb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
Yb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
f = lambda: L.mm(X, W[:, 0, :], Yb, epilogue="gelu", aux=Hb)  # noqa: E731
fl = 2.0 * T * n * h
res = {}
for rnd in range(2):
    for win in (30000, 250000, 0):
        for cap in (0, 2, 4, 8):
            fn(win)
            lib.ntp_gemm_set_split_k(cap)
            res.setdefault(f"win{win}_cap{cap}", []).append(round(fl / timed(f) / 1e9, 1))
fn(250000)
lib.ntp_gemm_set_split_k(1)
print(json.dumps(res, indent=0))
