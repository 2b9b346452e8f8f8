"""Planner timing (SURVEY §8(d) last row): the REFERENCE's build_shard_map +
build_reshard_plan (PRE and POST) + naive_contiguous_sync_volumes against this
package's C++ planner behind the same Python API, on the same triples, with
bit-equality of every output checked.  Build container only (imports the
reference read-only).  Writes profiles/r01_planner_timing.json."""

import json
import os
import sys
import time

sys.dont_write_bytecode = True
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(1, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from ntpsim import shardmap as R  # noqa: E402

from paper_2504_06095_b200 import shardmap as O  # noqa: E402


def best(fn, reps):
    t = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t = min(t, time.perf_counter() - t0)
    return t


def run(mod, k, n1, n2):
    s = mod.build_shard_map(k, n1, n2)
    pre = mod.build_reshard_plan(s, "pre_sync")
    post = mod.build_reshard_plan(s, "post_sync")
    nv = mod.naive_contiguous_sync_volumes(k, n1, n2)
    return s, pre, post, nv


def same(a, b):
    sa, pa, qa, na = a
    sb, pb, qb, nb = b
    if not (np.array_equal(sa.comp_rank, sb.comp_rank) and np.array_equal(sa.sync_rank, sb.sync_rank)):
        return False
    for x, y in ((pa, pb), (qa, qb)):
        if [(t.src, t.dst, tuple(t.cols)) for t in x.transfers] != \
           [(t.src, t.dst, tuple(t.cols)) for t in y.transfers]:
            return False
    return [list(map(tuple, r)) for r in na] == [list(map(tuple, r)) for r in nb]


def main():
    cases = [(4096, 4, 3), (14336, 4, 3), (14336, 4, 2), (8192, 8, 7), (12000, 32, 30),
             (1 << 20, 8, 5)]
    out = {"what": "reference ntpsim.shardmap planner vs paper_2504_06095_b200.shardmap (C++ "
                   "planner) -- build_shard_map + build_reshard_plan(pre, post) + "
                   "naive_contiguous_sync_volumes, best of N, 1 core", "cases": []}
    for k, n1, n2 in cases:
        reps = 3 if k > 100000 else 10
        ok = same(run(R, k, n1, n2), run(O, k, n1, n2))
        tr = best(lambda: run(R, k, n1, n2), reps)
        to = best(lambda: run(O, k, n1, n2), reps)
        out["cases"].append({"k": k, "n1": n1, "n2": n2, "identical": ok,
                             "reference_ms": round(tr * 1e3, 3), "ours_ms": round(to * 1e3, 3),
                             "speedup": round(tr / to, 1)})
        print(out["cases"][-1], flush=True)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "r01_planner_timing.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
