"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package ``ntpsim`` read-only from
/root/reference/pkg/src and records what the reference itself computes:

* shardmaps.json   -- build_shard_map / build_reshard_plan / naive overlaps /
                      attention_head_partition outputs (shardmap.py:141-260):
                      full arrays for small and anchor triples, sha256 digests
                      of the JSON forms for crit-02's 1000 random triples
                      (tests/test_acceptance.py:100-131 rng sequence).
* sync_cases.npz   -- nonuniform_grad_sync inputs and outputs (fp64, unit-major)
                      for crit-01-style instances (tests/test_acceptance.py:67-97)
                      with op sum and mean (tpnumerics.py:289-356), plus one
                      uniform_grad_sync case (tpnumerics.py:263-286).
* c1_digest.json   -- sha256 of the reference's C1 gradients before and after
                      nonuniform_grad_sync (h1024, k4096, TP4/TP3).
* golden_mlp.json   -- the reference's own frozen fixture (configs/golden_mlp.json).
* comm_comp_ratio.json -- perfmodel.comm_comp_ratio (perfmodel.py:244-278) values.

Nothing on the GPU box reads /root/reference: tests use only these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from ntpsim.shardmap import (  # noqa: E402
    POST_SYNC, PRE_SYNC, attention_head_partition, build_reshard_plan, build_shard_map,
    naive_contiguous_sync_volumes,
)
from ntpsim.tpnumerics import (  # noqa: E402
    MlpLayer, MlpReplica, assignment_from_comp, assignment_from_sync, contiguous_assignment,
    mlp_backward_tp, nonuniform_grad_sync, uniform_grad_sync,
)

OUT = os.path.dirname(os.path.abspath(__file__))


def digest_map(smap, pre, post) -> str:
    doc = {"map": smap.to_json_dict(), "pre": pre.to_json_dict(), "post": post.to_json_dict()}
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()


def units(rep):
    """Reference fragments -> unit-major [n_r, 2h] per rank (A col ; B row)."""
    return [np.concatenate([ga.T, gb], axis=1) for ga, gb in zip(rep.grad_a, rep.grad_b)]


def shardmaps():
    full = []
    for k, n1, n2 in [(8, 4, 4), (8, 4, 2), (12, 4, 3), (24, 6, 4), (60, 6, 3), (96, 8, 8),
                      (100, 7, 5), (100, 8, 6), (100, 5, 4), (37, 16, 1), (16, 4, 3),
                      (32, 4, 3), (16, 16, 15), (513, 16, 9), (4096, 4, 3), (12000, 32, 30)]:
        smap = build_shard_map(k, n1, n2)
        pre = build_reshard_plan(smap, PRE_SYNC)
        post = build_reshard_plan(smap, POST_SYNC)
        full.append({
            "k": k, "n1": n1, "n2": n2,
            "map": smap.to_json_dict(),
            "pre": pre.to_json_dict(), "post": post.to_json_dict(),
            "pre_stats": [pre.total_cols_moved, pre.max_cols_sent, pre.max_cols_received],
            "post_stats": [post.total_cols_moved, post.max_cols_sent, post.max_cols_received],
            "naive": [[list(p) for p in r] for r in naive_contiguous_sync_volumes(k, n1, n2)],
        })
    rng = np.random.default_rng(0)  # crit 02 sequence, test_acceptance.py:102-106
    crit02 = []
    for _ in range(1000):
        n1 = int(rng.integers(1, 17))
        n2 = int(rng.integers(1, n1 + 1))
        k = int(rng.integers(n1, 513))
        smap = build_shard_map(k, n1, n2)
        pre = build_reshard_plan(smap, PRE_SYNC)
        post = build_reshard_plan(smap, POST_SYNC)
        crit02.append([k, n1, n2, digest_map(smap, pre, post)])
    big = []
    for k, n1, n2 in [(14336, 4, 3), (14336, 4, 2), (8192, 4, 3), (8192, 2, 1), (14336, 8, 7)]:
        smap = build_shard_map(k, n1, n2)
        pre = build_reshard_plan(smap, PRE_SYNC)
        post = build_reshard_plan(smap, POST_SYNC)
        big.append({"k": k, "n1": n1, "n2": n2, "digest": digest_map(smap, pre, post),
                    "pre_stats": [pre.total_cols_moved, pre.max_cols_sent, pre.max_cols_received],
                    "naive": [[list(p) for p in r] for r in naive_contiguous_sync_volumes(k, n1, n2)]})
    heads = []
    for H, n in [(32, 3), (16, 3), (128, 32), (128, 30), (16, 16), (7, 2)]:
        counts, imb = attention_head_partition(H, n)
        heads.append({"heads": H, "n": n, "counts": counts.tolist(), "imbalance": imb})
    errors = []
    for k, n1, n2 in [(8, 4, 6), (3, 4, 2), (8, 0, 0), (0, 1, 1), (-1, 2, 1)]:
        try:
            build_shard_map(k, n1, n2)
            errors.append([k, n1, n2, None])
        except ValueError as e:
            errors.append([k, n1, n2, str(e)])
    with open(os.path.join(OUT, "shardmaps.json"), "w") as f:
        json.dump({"full": full, "crit02": crit02, "big": big, "heads": heads,
                   "errors": errors}, f, separators=(",", ":"))


def sync_cases():
    arrays = {}
    meta = []
    rng = np.random.default_rng(0)  # crit 01 sequence, test_acceptance.py:69-88
    picked = 0
    for inst in range(100):
        n1 = int(rng.integers(2, 17))
        n2 = int(rng.integers(1, n1 + 1))
        k = int(rng.integers(n1, 513))
        hidden = int(rng.integers(2, 7))
        seed = int(rng.integers(2**31))
        x1, x2 = rng.standard_normal((2, 4, hidden))
        g1, g2 = rng.standard_normal((2, 4, hidden))
        if k > 160 or picked >= 12:
            continue
        picked += 1
        for op in ("sum", "mean"):
            layer = MlpLayer.random(hidden, k, seed=seed)
            smap = build_shard_map(k, n1, n2)
            healthy = MlpReplica(layer, assignment_from_comp(smap))
            reduced = MlpReplica(layer, assignment_from_sync(smap))
            mlp_backward_tp(x1, healthy, g1)
            mlp_backward_tp(x2, reduced, g2)
            h_in, r_in = units(healthy), units(reduced)
            nonuniform_grad_sync(healthy, reduced, smap, op=op)
            h_out, r_out = units(healthy), units(reduced)
            tag = f"c{len(meta)}"
            meta.append({"tag": tag, "instance": inst, "k": k, "n1": n1, "n2": n2,
                         "hidden": hidden, "seed": seed, "op": op,
                         "h_counts": [len(c) for c in healthy.cols],
                         "r_counts": [len(c) for c in reduced.cols]})
            arrays[tag + "_x"] = np.stack([x1, x2])
            arrays[tag + "_g"] = np.stack([g1, g2])
            arrays[tag + "_h_in"] = np.concatenate(h_in).ravel()
            arrays[tag + "_r_in"] = np.concatenate(r_in).ravel()
            arrays[tag + "_h_out"] = np.concatenate(h_out).ravel()
            arrays[tag + "_r_out"] = np.concatenate(r_out).ravel()
    # one permuted-layout uniform sync (tests/test_tpnumerics.py:104-130 shape)
    k, hidden, n = 40, 4, 5
    layer = MlpLayer.random(hidden, k, seed=9)
    rng = np.random.default_rng(9)
    perm = rng.permutation(k)
    assignment = np.split(perm, np.sort(rng.choice(np.arange(1, k), n - 1, replace=False)))
    for op in ("sum", "mean"):
        reps = [MlpReplica(layer, assignment) for _ in range(3)]
        rng2 = np.random.default_rng(17)
        for rep in reps:
            mlp_backward_tp(rng2.standard_normal((2, hidden)), rep, rng2.standard_normal((2, hidden)))
        arrays[f"u_{op}_in"] = np.stack([np.concatenate(units(r)).ravel() for r in reps])
        uniform_grad_sync(reps, op=op)
        arrays[f"u_{op}_out"] = np.stack([np.concatenate(units(r)).ravel() for r in reps])
    arrays["u_cols"] = np.concatenate(assignment)
    arrays["u_counts"] = np.array([len(a) for a in assignment])
    np.savez_compressed(os.path.join(OUT, "sync_cases.npz"), **arrays)
    with open(os.path.join(OUT, "sync_cases.json"), "w") as f:
        json.dump({"cases": meta, "uniform": {"k": k, "hidden": hidden, "n": n, "replicas": 3,
                                              "layer_seed": 9, "grad_seed": 17}}, f, indent=1)


def c1_digest():
    """MlpLayer.random(1024, 4096, 0), map (4096,4,3), rng(0) draws."""
    layer = MlpLayer.random(1024, 4096, seed=0)
    smap = build_shard_map(4096, 4, 3)
    rng = np.random.default_rng(0)
    xh, gh = rng.standard_normal((4, 1024)), rng.standard_normal((4, 1024))
    xr, gr = rng.standard_normal((3, 1024)), rng.standard_normal((3, 1024))
    healthy = MlpReplica(layer, assignment_from_comp(smap))
    reduced = MlpReplica(layer, assignment_from_sync(smap))
    mlp_backward_tp(xh, healthy, gh)
    mlp_backward_tp(xr, reduced, gr)

    def dig(rep):
        h = hashlib.sha256()
        for u in units(rep):
            h.update(np.ascontiguousarray(u).tobytes())
        return h.hexdigest()

    doc = {"h_in": dig(healthy), "r_in": dig(reduced)}
    nonuniform_grad_sync(healthy, reduced, smap)
    doc.update({"h_out": dig(healthy), "r_out": dig(reduced)})
    with open(os.path.join(OUT, "c1_digest.json"), "w") as f:
        json.dump(doc, f, indent=1)


def comm_comp():
    """perfmodel.comm_comp_ratio (perfmodel.py:244-278): the reference's byte
    accounting of the busiest reshard rank over backward FLOPs."""
    from ntpsim.perfmodel import ModelShape, comm_comp_ratio
    cases = []
    for hidden, layers, heads, ffn in ((2048, 24, 16, 8192), (4096, 32, 32, 14336),
                                       (12288, 96, 96, None), (1024, 4, 8, 4096)):
        shape = ModelShape(hidden=hidden, layers=layers, heads=heads, ffn=ffn)
        for n1, n2, pp, lb, seq, b in ((4, 3, 1, 4, 2048, 2), (8, 6, 4, 2, 4096, 2),
                                       (4, 4, 1, 4, 2048, 2), (32, 30, 8, 1, 8192, 2),
                                       (8, 7, 2, 8, 1024, 4)):
            if n1 > heads:
                continue
            cases.append({"shape": [hidden, layers, heads, ffn], "n1": n1, "n2": n2, "pp": pp,
                          "local_batch": lb, "seq_len": seq, "bytes_per_element": b,
                          "ratio": comm_comp_ratio(shape, n1, n2, pp, lb, seq, b)})
    with open(os.path.join(OUT, "comm_comp_ratio.json"), "w") as f:
        json.dump(cases, f, indent=1)


if __name__ == "__main__":
    shutil.copy(os.path.join(REF, "ntpsim", "configs", "golden_mlp.json"),
                os.path.join(OUT, "golden_mlp.json"))
    shardmaps()
    sync_cases()
    c1_digest()
    comm_comp()
    print("fixtures written to", OUT)
