"""DP > 2 on one GPU (all R replicas in one HBM): the C3 shape -- DP=4 x TP2
with one replica at TP1 -- over the GPT-1.3B MLP gradients (24 x ffn 8192,
unit 2h, bf16), through ntp_multi_sync with the 128-bit-load and the TMA-bulk
kernels.  HBM roofline: 2 * R * S * b bytes per launch.  JSON out."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.plans import OPS, MultiPlan, layout_offsets  # noqa: E402
from paper_2504_06095_b200.shardmap import build_shard_map  # noqa: E402
from paper_2504_06095_b200.tpnumerics import assignment_from_comp, assignment_from_sync  # noqa: E402


def main():
    h, ffn, layers = 2048, 8192, 24
    k, unit = ffn * layers, 2 * h
    smap = build_shard_map(k, 2, 1)
    layouts = [assignment_from_comp(smap)] * 3 + [assignment_from_sync(smap)]
    w = np.array([2, 2, 2, 1], dtype=np.float64) / 7
    bufs, offs, arenas, base = [], [], [], 0
    g = torch.Generator(device="cuda").manual_seed(0)
    for cols in layouts:
        owner, off = layout_offsets(cols, k, unit)
        bufs.append(owner + base)
        offs.append(off)
        for c in cols:
            arenas.append(torch.randn(len(c) * unit, generator=g, device="cuda").to(torch.bfloat16))
        base += len(cols)
    plan = MultiPlan(_lib.NTP_BF16, 4).add_units(unit, bufs, offs).finalize().upload(0)
    ptrs = [a.data_ptr() for a in arenas]
    L = _lib.load()
    nbytes = 2 * 4 * k * unit * 2
    out = {"workload": "C3 shape on one GPU: 3 x TP2 + 1 x TP1 replicas, GPT-1.3B MLP grads, bf16",
           "bytes_per_launch": nbytes, "chunks": plan.n_chunks}
    peak = 6541.8
    for variant, name in ((1, "ldg"), (2, "bulk")):
        L.ntp_multi_set_kernel(variant)
        for _ in range(3):
            plan.sync(ptrs, OPS["weighted"], w)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            plan.sync(ptrs, OPS["weighted"], w)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out[name] = {"ms": round(ms, 3), "GBps": round(nbytes / ms / 1e6, 1),
                     "hbm_frac": round(nbytes / ms / 1e6 / peak, 3)}
    L.ntp_multi_set_kernel(0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
