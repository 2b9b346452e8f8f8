"""Per-item epilogue timestamps of one GEMM launch (debug hook
ntp_gemm_debug_trace) with split-K off and on: where does the tail go?"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib, linear as L  # noqa: E402

lib = _lib.load()
T, h, n = 8192, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 4779
which = sys.argv[2] if len(sys.argv) > 2 else "wgrad"
npad = (n + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
G = torch.randn((T, h), generator=g, device="cuda").to(torch.bfloat16)
W = torch.randn((n, 2, h), generator=g, device="cuda").to(torch.bfloat16)
Hb = torch.empty((T, npad), dtype=torch.bfloat16, device="cuda")[:, :n]
Yb = torch.randn((T, npad), generator=g, device="cuda").to(torch.bfloat16)[:, :n]
grads = torch.empty((n, 2, h), dtype=torch.bfloat16, device="cuda")
fn = {"wgrad": lambda: L.mm(Yb.T, G.T, grads[:, 1, :]),
      "fwd1": lambda: L.mm(X, W[:, 0, :], Yb, epilogue="gelu", aux=Hb)}[which]
buf = torch.zeros(148 * 16 * 8, dtype=torch.int64, device="cuda")
res = {}
for cap in (0, 2, 8):
    lib.ntp_gemm_set_split_k(cap)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    buf.zero_()
    lib.ntp_gemm_debug_trace(ctypes.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    lib.ntp_gemm_debug_trace(None)
    tr = buf.view(148, 16, 8).cpu()
    t0 = int(tr[:, 0, 3][tr[:, 0, 3] > 0].min())
    rows = []
    for b in range(0, 148, 2):  # leader CTAs
        for loc in range(16):
            it, tf, td = (int(x) for x in tr[b, loc, :3])
            if tf == 0:
                break
            rows.append((b // 2, loc, it, (tf - t0) / 1e3, (td - t0) / 1e3))
    end = max(r[4] for r in rows)
    # leader-CTA pipeline marks of the last item (relative us)
    lastloc = {}
    for b in range(0, 148, 2):
        for loc in range(15, -1, -1):
            if int(tr[b, loc, 1]):
                v = [(int(x) - t0) / 1e3 if int(x) else None for x in tr[b, loc, 4:8]]
                prev = [(int(x) - t0) / 1e3 if int(x) else None for x in tr[b, loc - 1, [1, 2, 4, 5, 6, 7]]] if loc else None
                lastloc[b // 2] = {"loc": loc, "item": int(tr[b, loc, 0]),
                                   "prod_first,prod_last,mma_first,mma_last": [round(x, 1) if x else x for x in v],
                                   "full,done": [round((int(tr[b, loc, 1]) - t0) / 1e3, 1), round((int(tr[b, loc, 2]) - t0) / 1e3, 1)],
                                   "prev full,done,pf,pl,mf,ml": [round(x, 1) if x else x for x in prev] if prev else None}
                break
    last = sorted(rows, key=lambda r: -r[4])[:6]
    per_loc = {}
    for r in rows:
        per_loc.setdefault(r[1], []).append(r[4] - r[3])
    res[cap] = {"span_us": end,
                "start_spread_us": (int(tr[:, 0, 3].max()) - t0) / 1e3,
                "epi_us_by_local": {k: [round(min(v), 2), round(max(v), 2)] for k, v in per_loc.items()},
                "full_time_by_local_us": {loc: [round(min(r[3] for r in rows if r[1] == loc), 1),
                                                round(max(r[3] for r in rows if r[1] == loc), 1)]
                                          for loc in per_loc},
                "last_items": {k: lastloc[k] for k in list(lastloc)[:4] + list(lastloc)[-4:]},
                "last_finishers": [[r[0], r[1], r[2], round(r[3], 1), round(r[4], 1)] for r in last]}
lib.ntp_gemm_set_split_k(1)
print(json.dumps(res, indent=1))
