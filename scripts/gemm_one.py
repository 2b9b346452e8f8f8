"""Run one C4 per-rank GEMM a few times (for ncu).  usage: gemm_one.py {fwd1,fwd2,wgrad} [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import linear as L  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fwd2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
T, h, n = 8192, 4096, 4779
npad = (n + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
H = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
Y = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
Z = torch.empty((T, h), dtype=torch.float32, device="cuda")
grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
for _ in range(iters):
    if which == "fwd1":
        L.mm(X, W[:, 0, :], Y, epilogue="gelu", aux=H)
    elif which == "fwd2":
        L.mm(Y, W[:, 1, :].T, Z)
    else:
        L.mm(Y.T, G.T, grads[:, 1, :])
torch.cuda.synchronize()
print("ok", which)
