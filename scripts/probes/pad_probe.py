"""Which GEMM writes into its output's pitch padding?  (debug probe)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.linear import MlpShard, _pad8, mm  # noqa: E402

L = _lib.load()
h, T = 512, 384
for n in (4779, 4781, 600, 601, 3584, 100):
    for split in (1, 0):
        L.ntp_gemm_set_split_k(split)
        rng = np.random.default_rng(n)
        A = rng.standard_normal((h, n)) / np.sqrt(h)
        B = rng.standard_normal((n, h)) / np.sqrt(n)
        sh = MlpShard(A, B, np.arange(n))
        X = torch.randn((T, h), device="cuda").to(torch.bfloat16)
        G = torch.randn((T, h), device="cuda").to(torch.bfloat16)
        npad = _pad8(n) + 8
        res = {}
        for name in ("gelu", "dgelu"):
            Hb = torch.full((T, npad), float("nan"), device="cuda").to(torch.bfloat16)
            Yb = torch.full((T, npad), float("nan"), device="cuda").to(torch.bfloat16)
            H, Y = Hb[:, :n], Yb[:, :n]
            mm(X, sh.W[:, 0, :], Y, epilogue="gelu", aux=H)
            if name == "dgelu":
                Db = torch.full((T, npad), float("nan"), device="cuda").to(torch.bfloat16)
                mm(G, sh.W[:, 1, :], Db[:, :n], epilogue="dgelu", aux=H)
                bufs = {"D": Db}
            else:
                bufs = {"H": Hb, "Y": Yb}
            torch.cuda.synchronize()
            for k, b in bufs.items():
                pad = b[:, n:]
                bad = ~torch.isnan(pad.float())
                res[k] = (int(bad.sum()), bad.nonzero()[:3].tolist())
        print(n, "split", split, res, flush=True)
L.ntp_gemm_set_split_k(1)
