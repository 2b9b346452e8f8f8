"""Compare the sync kernel variants on the 1-GPU C2 workload (device time,
bitwise agreement).  Usage: python scripts/sync_variants.py [steps]"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.plans import OPS, tensor_ptrs  # noqa: E402
from paper_2504_06095_b200.workloads import SHAPES, build_plan, pair_layout  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    workload = sys.argv[2] if len(sys.argv) > 2 else "gpt-1.3b"
    L = _lib.load()
    torch.cuda.set_device(0)
    lay = pair_layout(SHAPES[workload], 4, 3)
    plan = build_plan(lay, torch.bfloat16).upload(0)
    gen = torch.Generator(device="cuda").manual_seed(0)
    init = [torch.randn(e, generator=gen, device="cuda").to(torch.bfloat16)
            for e in lay.h_elems + lay.r_elems]
    results = {}
    ref = None
    for name, v in (("ldg", 1), ("bulk4x1", 2), ("bulk3x2", 3)):
        _lib.check(L.ntp_set_option(0, v))
        arenas = [t.clone() for t in init]
        ptrs = tensor_ptrs(arenas)
        plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
        torch.cuda.synchronize()
        out = torch.cat([a.view(-1) for a in arenas])
        if ref is None:
            ref = out
        same = bool(torch.equal(out, ref))
        for _ in range(5):
            plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            plan.grad_sync(ptrs, OPS["weighted"], 4 / 7, 3 / 7)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        gbs = 4 * lay.elems * 2 / (ms * 1e-3) / 1e9
        results[name] = {"ms": round(ms, 4), "hbm_gbs": round(gbs, 1),
                         "frac_of_6541.8": round(gbs / 6541.8, 4), "bitwise_equal_to_ldg": same}
        del arenas
        torch.cuda.empty_cache()
    _lib.check(L.ntp_set_option(0, 0))
    # reference point: torch copy of the same byte volume (2 x 4.8 GB read+write)
    src = torch.cat([t.view(-1) for t in init])
    dst = torch.empty_like(src)
    for _ in range(3):
        dst.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        dst.copy_(src)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    results["torch_copy_same_bytes"] = {"ms_per_2x": round(2 * ms, 4),
                                        "hbm_gbs": round(2 * src.numel() * 2 / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps({"workload": workload, "steps": steps, "variants": results}, indent=1))


if __name__ == "__main__":
    main()
