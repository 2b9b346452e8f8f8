"""Time the REFERENCE's own Python nonuniform_grad_sync in this container (it
cannot travel to the GPU box), on the C1 config and on one layer of the C2
workload's MLP -- the reference has no attention gradients.  Writes
profiles/r01_reference_python_timing.json.  Build container only."""

import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
from ntpsim.shardmap import build_shard_map  # noqa: E402
from ntpsim.tpnumerics import (  # noqa: E402
    MlpLayer, MlpReplica, assignment_from_comp, assignment_from_sync, nonuniform_grad_sync,
)


def time_case(hidden, k, n1, n2, reps=3):
    layer = MlpLayer(np.zeros((hidden, k)), np.zeros((k, hidden)))
    smap = build_shard_map(k, n1, n2)
    rng = np.random.default_rng(0)
    best = float("inf")
    for _ in range(reps):
        h = MlpReplica(layer, assignment_from_comp(smap))
        r = MlpReplica(layer, assignment_from_sync(smap))
        h.grad_a = [rng.standard_normal(a.shape) for a in h.a_frags]
        h.grad_b = [rng.standard_normal(b.shape) for b in h.b_frags]
        r.grad_a = [rng.standard_normal(a.shape) for a in r.a_frags]
        r.grad_b = [rng.standard_normal(b.shape) for b in r.b_frags]
        t0 = time.perf_counter()
        nonuniform_grad_sync(h, r, smap)
        best = min(best, time.perf_counter() - t0)
    elems = 2 * hidden * k
    return {"hidden": hidden, "k": k, "n1": n1, "n2": n2, "seconds_best_of_3": round(best, 4),
            "elements_per_replica": elems,
            "synced_gradient_GBps_as_bf16": round(elems * 2 / best / 1e9, 4),
            "synced_gradient_GBps_as_f64": round(elems * 8 / best / 1e9, 4)}


if __name__ == "__main__":
    out = {"what": "reference ntpsim.tpnumerics.nonuniform_grad_sync (pure Python + numpy, "
                   "1 core), timed in the build container",
           "cpu": os.popen("grep -m1 'model name' /proc/cpuinfo").read().strip(),
           "cases": [time_case(1024, 4096, 4, 3), time_case(2048, 8192, 4, 3)]}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "r01_reference_python_timing.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))
