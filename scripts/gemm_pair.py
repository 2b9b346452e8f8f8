"""The C4 per-rank GEMMs through ours and through cuBLAS (padded contiguous
operands), a few launches each -- for ncu side-by-side captures (e.g. at
base clocks, so kernel efficiency is compared without the power cap).

    python scripts/gemm_pair.py [which,...|all] [iters] [n_i]
    NTP_GEMM_EPI_SLEEP=0|1, NTP_GEMM_RASTER=n, NTP_GEMM_DEBUG=bits select debug variants
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200 import linear as L  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4779
kinds = ["fwd1", "fwd2", "dgelu", "wgrad"] if which == "all" else which.split(",")
lib = _lib.load()
if "NTP_GEMM_EPI_SLEEP" in os.environ:
    lib.ntp_gemm_debug_epi_sleep.argtypes = [ctypes.c_int]
    lib.ntp_gemm_debug_epi_sleep(int(os.environ["NTP_GEMM_EPI_SLEEP"]))
if "NTP_GEMM_DEBUG" in os.environ:
    lib.ntp_gemm_debug_mode.argtypes = [ctypes.c_int]
    lib.ntp_gemm_debug_mode(int(os.environ["NTP_GEMM_DEBUG"]))
if "NTP_GEMM_RASTER" in os.environ:
    lib.ntp_gemm_debug_raster.argtypes = [ctypes.c_int]
    lib.ntp_gemm_debug_raster(int(os.environ["NTP_GEMM_RASTER"]))
T, h = 8192, 4096
npad = (n + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
Wc = torch.randn((npad, h), generator=g, device="cuda").to(torch.bfloat16)
H = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)
Y = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)
D = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")
Z = torch.empty((T, h), dtype=torch.float32, device="cuda")
grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
for _ in range(iters):
    for k in kinds:
        if k == "fwd1":
            L.mm(X, W[:, 0, :], Y[:, :n], epilogue="gelu", aux=H[:, :n])
            torch.matmul(X, Wc.T)
        elif k == "fwd2":
            L.mm(Y[:, :n], W[:, 1, :].T, Z)
            torch.matmul(Y, Wc)
        elif k == "dgelu":
            L.mm(G, W[:, 1, :], D[:, :n], epilogue="dgelu", aux=H[:, :n])
            torch.matmul(G, Wc.T)
        else:
            L.mm(Y[:, :n].T, G.T, grads[:, 1, :])
            torch.matmul(Y.T, G)
torch.cuda.synchronize()
print("ok", which)
