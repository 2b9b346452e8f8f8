"""L2 cache policy of the bulk sync kernel's copies (NTP_OPT_SYNC_L2: 0 none,
1 loads evict_first, 2 loads + stores evict_first) on the N=1 bench
workloads: C1 after a 256 MB L2 write-flush (the bench's timing rule: the
flush leaves dirty lines the kernel must evict) and C2 (4.8 GB, no flush).
Per-step CUDA events, median of `steps`.  Usage: python scripts/l2_hint_probe.py [steps]"""

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
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    L = _lib.load()
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    hbm = bench.peaks()["hbm_gbs"]
    out = {}
    for wl, do_flush in (("mlp-h1024-ffn4096", True), ("gpt-1.3b", False)):
        dt = bench._torch_dtype(wl)
        eb = bench.ELEM_BYTES[bench.WORKLOADS[wl][4]]
        lay = pair_layout(SHAPES[wl], 4, 3)
        plan = build_plan(lay, dt).upload(0)
        arenas = [torch.randn(e, device="cuda").to(dt) for e in lay.h_elems + lay.r_elems]
        ptrs = tensor_ptrs(arenas)
        for hint in (0, 1, 2, 0):
            _lib.check(L.ntp_set_option(3, hint))
            _lib.check(L.ntp_set_option(0, 2))  # the bulk kernel (C1's AUTO choice too)
            for _ in range(3):
                plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
            torch.cuda.synchronize()
            for i in range(steps):
                if do_flush:
                    flush.fill_(i & 0xFF)
                ev[2 * i].record()
                plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
                ev[2 * i + 1].record()
            torch.cuda.synchronize()
            ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps))
            med = ts[len(ts) // 2]
            out.setdefault(wl, []).append(
                {"l2_hint": hint, "us_median": round(med * 1e3, 2),
                 "frac_hbm": round(4 * lay.elems * eb / (med * 1e-3) / 1e9 / hbm, 4)})
        del arenas
        torch.cuda.empty_cache()
    _lib.check(L.ntp_set_option(3, 0))
    _lib.check(L.ntp_set_option(0, 0))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
