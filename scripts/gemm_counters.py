"""Where the tcgen05 GEMM's MMA issuer waits: per-CTA clock64 counters of the
MMA warp's full-stage and free-accumulator waits and the MMA loop's total, on the C4 per-rank GEMMs (debug hook
ntp_gemm_debug_counters).  Prints one JSON line per GEMM.

    [NTP_GEMM_RASTER=g] [NTP_GEMM_L2PROMO=0..3] python scripts/gemm_counters.py [n_i]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200 import linear as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4779
lib = _lib.load()
lib.ntp_gemm_debug_counters.argtypes = [ctypes.c_void_p]
for var, fn in (("NTP_GEMM_RASTER", "ntp_gemm_debug_raster"), ("NTP_GEMM_L2PROMO", "ntp_gemm_debug_l2promo")):
    if var in os.environ:
        getattr(lib, fn).argtypes = [ctypes.c_int]
        getattr(lib, fn)(int(os.environ[var]))
tag = os.environ.get("TAG", "")
T, h = 8192, 4096
npad = (n + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
H = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)
Y = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)
D = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")
Z = torch.empty((T, h), dtype=torch.float32, device="cuda")
grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
cases = {
    "fwd1": lambda: L.mm(X, W[:, 0, :], Y[:, :n], epilogue="gelu", aux=H[:, :n]),
    "fwd2": lambda: L.mm(Y[:, :n], W[:, 1, :].T, Z),
    "dgelu": lambda: L.mm(G, W[:, 1, :], D[:, :n], epilogue="dgelu", aux=H[:, :n]),
    "wgrad": lambda: L.mm(Y[:, :n].T, G.T, grads[:, 1, :]),
}
buf = torch.zeros(148 * 4, dtype=torch.int64, device="cuda")
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    buf.zero_()
    lib.ntp_gemm_debug_counters(ctypes.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    lib.ntp_gemm_debug_counters(None)
    c = buf.view(148, 4).cpu().double()
    lead = c[0::2]  # leader CTAs run the MMA warp
    tot = lead[:, 3].mean().item()
    print(json.dumps({"tag": tag, "gemm": name, "n_i": n, "mma_loop_kcycles": round(tot / 1e3, 1),
                      "mma_wait_full_frac": round((lead[:, 1] / lead[:, 3]).mean().item(), 4),
                      "mma_wait_acc_frac": round((lead[:, 2] / lead[:, 3]).mean().item(), 4)}),
          flush=True)
