"""Sync kernel variants on a small (L2-sized) workload, 1 GPU, L2 flushed
before every timed step: which kernel AUTO should pick below the bulk
threshold.  Usage: python scripts/small_variants.py [workload steps]"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.plans import OPS, tensor_ptrs  # noqa: E402
from paper_2504_06095_b200.workloads import SHAPES, build_plan, pair_layout  # noqa: E402


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "mlp-h1024-ffn4096"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    L = _lib.load()
    torch.cuda.set_device(0)
    dtype = bench._torch_dtype(workload)
    eb = bench.ELEM_BYTES[bench.WORKLOADS[workload][4]]
    lay = pair_layout(SHAPES[workload], 4, 3)
    plans = {}
    for mc in (1184, 4096, 8192, 16384):  # NTP_OPT_PLAN_MIN_CHUNKS
        _lib.check(L.ntp_set_option(2, mc))
        plans[mc] = build_plan(lay, dtype).upload(0)
    _lib.check(L.ntp_set_option(2, 1184))
    plan = plans[1184]
    arenas = [torch.randn(e, device="cuda").to(dtype) for e in lay.h_elems + lay.r_elems]
    ptrs = tensor_ptrs(arenas)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    hbm = bench.peaks()["hbm_gbs"]
    out = {"workload": workload, "chunks": plan.stats["n_chunks"], "bytes": 4 * lay.elems * eb}
    for name, v, cap in (("auto", 0, 0), ("ldg", 1, 0), ("bulk4x1", 2, 0), ("bulk3x2", 3, 0),
                         ("ldg_cap296", 1, 296), ("ldg_cap592", 1, 592)):
        _lib.check(L.ntp_set_option(0, v))
        _lib.check(L.ntp_set_option(1, cap))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
        for _ in range(5):
            plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
        torch.cuda.synchronize()
        for i in range(steps):
            flush.fill_(i & 0xFF)
            ev[2 * i].record()
            plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
            ev[2 * i + 1].record()
        torch.cuda.synchronize()
        ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps))
        med = ts[len(ts) // 2]
        out[name] = {"us_median": round(med * 1e3, 2), "us_min": round(ts[0] * 1e3, 2),
                     "frac_hbm": round(4 * lay.elems * eb / (med * 1e-3) / 1e9 / hbm, 4)}
    _lib.check(L.ntp_set_option(0, 0))
    _lib.check(L.ntp_set_option(1, 0))
    for mc, pl in plans.items():  # AUTO kernel, smaller chunks
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
        for i in range(steps):
            flush.fill_(i & 0xFF)
            ev[2 * i].record()
            pl.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
            ev[2 * i + 1].record()
        torch.cuda.synchronize()
        ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps))
        out[f"auto_min_chunks_{mc}"] = {"chunks": pl.stats["n_chunks"],
                                        "us_median": round(ts[len(ts) // 2] * 1e3, 2)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
