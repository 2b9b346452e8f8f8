"""NVLink bytes of the N=2 bench step, per GPU and direction, from ncu.

The bench's N>1 kernels are signalled (they wait for the partner process), so
ncu cannot replay them on their own.  This script runs the SAME per-process
plans (dist.process_plan_units, executor policy "split", the GPT-1.3B C2
workload with bench.py's N=2 placement: healthy TP4 on GPU 0, reduced TP3 on
GPU 1) from ONE process over peer-enabled GPUs, unsignalled: GPU 0 runs rank
0's plan, then GPU 1 runs rank 1's.  Under

    ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum,gpu__time_duration.sum python scripts/nvlink_traffic.py \\
        [workload reps world plan.json]

each kernel reports its own GPU's NVLink TX / RX bytes.  With two GPUs one
link pair carries everything, so during the real (concurrent) step
GPU 0's TX = kernel0.nvltx + kernel1.nvlrx and GPU 0's RX = kernel0.nvlrx +
kernel1.nvltx (and the mirror for GPU 1); scripts/nvlink_traffic_summary.py
turns the ncu CSV into those per-direction totals.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

from paper_2504_06095_b200 import _lib  # noqa: E402
from paper_2504_06095_b200.dist import Placement, process_plan_units  # noqa: E402
from paper_2504_06095_b200.plans import OPS, Plan, dtype_code  # noqa: E402
from paper_2504_06095_b200.workloads import SHAPES, pair_layout  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    world = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    plan_out = sys.argv[4] if len(sys.argv) > 4 else None
    _lib.load()
    for a in range(world):
        rt.cudaSetDevice(a)
        for b in range(world):
            if a != b:
                rt.cudaDeviceEnablePeerAccess(b, 0)
    dtype = torch.bfloat16
    eb = 2
    lay = pair_layout(SHAPES[name], 4, 3)
    plc = Placement.default(world, 4, 3)
    elems = list(lay.h_elems) + list(lay.r_elems)
    arenas = {s: torch.randn(elems[s], device=f"cuda:{plc.proc_of_slot(s)}").to(dtype)
              for s in range(len(elems))}
    plans = []
    # algorithmic NVLink bytes of each rank's plan, per peer GPU: a unit executed
    # on `rank` whose other copy lives on GPU q reads unit*eb from q and writes
    # unit*eb to q
    per_peer = {r: {q: 0 for q in range(world)} for r in range(world)}
    for rank in range(world):
        units, touched = process_plan_units(lay, plc, rank, "split")
        if not units:
            continue
        order = sorted(touched)
        remap = np.full(len(elems), -1, dtype=np.int64)
        for i, s in enumerate(order):
            remap[s] = i
        p = Plan(dtype_code(dtype))
        for unit, hs, ho, rs, ro in units:
            p.add_units(unit, remap[hs], ho, remap[rs], ro)
            for slots in (hs, rs):
                procs = np.array([plc.proc_of_slot(int(x)) for x in range(len(elems))])[slots]
                for q in np.unique(procs):
                    if q != rank:
                        per_peer[rank][int(q)] += int((procs == q).sum()) * unit * eb
        plans.append((rank, p.finalize().upload(rank), [arenas[s].data_ptr() for s in order]))
    if plan_out:
        import json
        with open(plan_out, "w") as f:
            json.dump({"world": world, "workload": name,
                       "read_and_write_bytes_per_peer": {str(r): {str(q): v for q, v in d.items()}
                                                         for r, d in per_peer.items()}}, f)
    for _ in range(reps):
        for rank, p, bufs in plans:
            with torch.cuda.device(rank):
                p.grad_sync(bufs, OPS["weighted"], 4 / 7, 3 / 7, torch.cuda.current_stream(rank))
                torch.cuda.synchronize(rank)
    print("nvlink_traffic done", flush=True)


if __name__ == "__main__":
    main()
