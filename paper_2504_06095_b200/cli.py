"""Command line with the reference's ``shardmap`` and ``verify`` subcommands.

    python -m paper_2504_06095_b200.cli shardmap --k K --n1 N1 --n2 N2 [--json]
    python -m paper_2504_06095_b200.cli verify [--suite S] [--seed N] [--json]

Same flags, output lines, JSON shapes and exit codes as ``ntpsim`` (cli.py:
328-382, 885-928): 0 ok, 1 failed verification, 2 bad arguments (``error: ...``
on stderr).  ``verify`` runs the reference's oracle suites against THIS
implementation: the shard algebra through the C planner, and the gradient
syncs through the device kernels (a GPU is required for those suites).
The simulator subcommands (``simulate``, ``calibrate``) are out of scope.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import __version__
from .shardmap import (
    POST_SYNC, PRE_SYNC, apply_plan, build_reshard_plan, build_shard_map,
    naive_contiguous_sync_volumes,
)


def _rel_err(got, want) -> float:
    """cli.py:83-87."""
    denom = np.linalg.norm(want)
    if denom == 0.0:
        return float(np.linalg.norm(got))
    return float(np.linalg.norm(np.asarray(got) - np.asarray(want)) / denom)


def _ok(name, detail):
    return {"name": name, "passed": True, "detail": detail, "case": None}


def _fail(name, detail, case):
    return {"name": name, "passed": False, "detail": detail, "case": case}


def _suite_shard_invariants(seed: int) -> dict:
    """cli.py:90-161 against the C planner."""
    rng = np.random.default_rng(seed)
    for i in range(1000):
        n1 = int(rng.integers(1, 17))
        n2 = int(rng.integers(1, n1 + 1))
        k = int(rng.integers(n1, 513))
        case = {"instance": i, "k": k, "n1": n1, "n2": n2}
        smap = build_shard_map(k, n1, n2)
        comp = np.concatenate([smap.comp_columns(r) for r in range(n1)])
        sync = np.concatenate([smap.sync_columns(r) for r in range(n2)])
        if not (np.array_equal(np.sort(comp), np.arange(k))
                and np.array_equal(np.sort(sync), np.arange(k))):
            return _fail("shard-invariants", "columns not partitioned exactly once", case)
        cc, sc = smap.comp_counts(), smap.sync_counts()
        if not all(k // n1 <= c <= -(-k // n1) for c in cc):
            return _fail("shard-invariants", "comp shard sizes not balanced within 1", case)
        if not all(k // n2 <= c <= -(-k // n2) for c in sc):
            return _fail("shard-invariants", "sync shard sizes not balanced within 1", case)
        if np.any(np.diff(smap.sync_rank) < 0):
            return _fail("shard-invariants", "sync shard not contiguous", case)
        post = build_reshard_plan(smap, POST_SYNC)
        links = post.link_volumes()
        for src in range(n2):
            vols = [links.get((src, dst), 0) for dst in range(n2, n1)]
            if vols and max(vols) - min(vols) > 1:
                return _fail("shard-invariants", f"offload links from sync rank {src} unbalanced", case)
        pre = build_reshard_plan(smap, PRE_SYNC)
        if not np.array_equal(apply_plan(smap.comp_rank, pre), smap.sync_rank):
            return _fail("shard-invariants", "pre-sync plan does not reach sync layout", case)
        if not np.array_equal(apply_plan(smap.sync_rank, post), smap.comp_rank):
            return _fail("shard-invariants", "post-sync plan does not restore comp layout", case)
        again = build_shard_map(k, n1, n2)
        if not (np.array_equal(again.comp_rank, smap.comp_rank)
                and np.array_equal(again.sync_rank, smap.sync_rank)):
            return _fail("shard-invariants", "rebuild is not deterministic", case)
    case = {"k": 12000, "n1": 32, "n2": 30}
    smap = build_shard_map(12000, 32, 30)
    if set(smap.comp_counts().tolist()) != {375} or set(smap.sync_counts().tolist()) != {400}:
        return _fail("shard-invariants", "contrast-case shard sizes differ from 375/400", case)
    sizes = {s for r in naive_contiguous_sync_volumes(12000, 32, 30) for _, s in r}
    if min(sizes) != 25 or max(sizes) != 375:
        return _fail("shard-invariants", "naive contiguous splits do not span 25..375", case)
    post = build_reshard_plan(smap, POST_SYNC)
    stats = (post.total_cols_moved, post.max_cols_sent, post.max_cols_received)
    if stats != (750, 25, 375):
        return _fail("shard-invariants", f"contrast-case plan stats {stats}, expected (750, 25, 375)", case)
    return _ok("shard-invariants", "1000 random triples + contrast case")


def _suite_tp_numerics(seed: int) -> dict:
    """cli.py:164-247: 100 nonuniform syncs (fp64, on the device) equal dense
    sums, 10 permuted-layout uniform syncs, 10 head-sharded attention forwards."""
    import torch

    from . import tpnumerics as T
    if not torch.cuda.is_available():
        return _fail("tp-numerics", "needs a CUDA device (no CPU fallback)", {})
    rng = np.random.default_rng(seed)
    start = time.time()
    worst = 0.0
    for i in range(100):
        n1 = int(rng.integers(2, 17))
        n2 = int(rng.integers(1, n1 + 1))
        k = int(rng.integers(n1, 513))
        hidden = int(rng.integers(2, 7))
        case = {"instance": i, "k": k, "n1": n1, "n2": n2, "hidden": hidden}
        layer = T.MlpLayer.random(hidden, k, seed=int(rng.integers(2**31)))
        smap = build_shard_map(k, n1, n2)
        h = T.MlpReplica(layer, T.assignment_from_comp(smap), dtype=torch.float64)
        r = T.MlpReplica(layer, T.assignment_from_sync(smap), dtype=torch.float64)
        batch = int(rng.integers(2, 5))
        x1, x2, g1, g2 = (rng.standard_normal((batch, hidden)) for _ in range(4))
        T.mlp_backward_tp(x1, h, g1)
        T.mlp_backward_tp(x2, r, g2)
        d1 = T.MlpReplica(layer, [np.arange(k)], dtype=torch.float64)
        d2 = T.MlpReplica(layer, [np.arange(k)], dtype=torch.float64)
        T.mlp_backward_tp(x1, d1, g1)
        T.mlp_backward_tp(x2, d2, g2)
        T.nonuniform_grad_sync(h, r, smap)
        da = d1.dense_grads()[0] + d2.dense_grads()[0]
        db = d1.dense_grads()[1] + d2.dense_grads()[1]
        for rep in (h, r):
            ra, rb = rep.dense_grads()
            err = max(_rel_err(ra, da), _rel_err(rb, db))
            worst = max(worst, err)
            if err > 1e-12:
                case["rel_err"] = err
                return _fail("tp-numerics", "sync result differs from dense sum", case)
    for i in range(10):
        k = int(rng.integers(6, 65))
        hidden = int(rng.integers(2, 6))
        layer = T.MlpLayer.random(hidden, k, seed=int(rng.integers(2**31)))
        n = int(rng.integers(2, 7))
        perm = rng.permutation(k)
        assignment = np.split(perm, np.sort(rng.choice(np.arange(1, k), size=n - 1, replace=False)))
        reps, want_a, want_b = [], 0.0, 0.0
        for _ in range(3):
            rep = T.MlpReplica(layer, assignment, dtype=torch.float64)
            x = rng.standard_normal((3, hidden))
            g = rng.standard_normal((3, hidden))
            T.mlp_backward_tp(x, rep, g)
            da, db = rep.dense_grads()
            want_a, want_b = want_a + da, want_b + db
            reps.append(rep)
        T.uniform_grad_sync(reps)
        for rep in reps:
            ra, rb = rep.dense_grads()
            err = max(_rel_err(ra, want_a), _rel_err(rb, want_b))
            worst = max(worst, err)
            if err > 1e-12:
                return _fail("tp-numerics", "uniform sync not invariant to shard permutation",
                             {"instance": i, "k": k, "n": n, "rel_err": err})
    for i in range(10):  # head-sharded attention forward == dense (same rng stream)
        heads = int(rng.integers(2, 9))
        head_dim = int(rng.integers(2, 5))
        hidden = int(rng.integers(3, 7))
        n = int(rng.integers(1, heads + 1))
        att = T.AttentionLayer.random(heads, hidden, head_dim, seed=int(rng.integers(2**31)))
        rep = T.AttentionReplica(att, T.contiguous_assignment(heads, n), dtype=torch.float64)
        x = rng.standard_normal((4, hidden))
        err = _rel_err(T.attention_forward_tp(x, rep), T.attention_forward_dense(x, att))
        worst = max(worst, err)
        if err > 1e-12:
            return _fail("tp-numerics", "sharded attention differs from dense",
                         {"instance": i, "heads": heads, "n": n, "rel_err": err})
    elapsed = time.time() - start
    if elapsed > 30.0:
        return _fail("tp-numerics", f"suite exceeded 30 s budget ({elapsed:.1f} s)", {})
    return _ok("tp-numerics", f"120 instances, worst rel err {worst:.2e}, {elapsed:.1f} s")


def _central_differences(T, x, g, A, B, h: float = 1e-6):
    """d(sum(Z * g))/dA and /dB by central differences, every entry at once:
    the +h / -h bumps of all hidden*ffn entries of A (then of B) form one batch
    of perturbed weight matrices evaluated by a single batched fp64 forward."""
    import torch
    dev = T._device()
    X, G = T._dev64(x), T._dev64(g)
    A, B = T._dev64(A), T._dev64(B)

    def losses(As, Bs):  # As [n, h, f], Bs [n, f, h] -> [n]
        Z = torch.matmul(T._gelu_t(torch.matmul(X, As)), Bs)
        return (Z * G).sum(dim=(1, 2))
    out = []
    for W, other, first in ((A, B, True), (B, A, False)):
        n = W.numel()
        eye = torch.eye(n, dtype=torch.float64, device=dev).reshape(n, *W.shape) * h
        Wp, Wm = W.unsqueeze(0) + eye, W.unsqueeze(0) - eye
        O = other.unsqueeze(0).expand(n, *other.shape)
        up = losses(Wp, O) if first else losses(O, Wp)
        dn = losses(Wm, O) if first else losses(O, Wm)
        out.append(((up - dn) / (2 * h)).reshape(W.shape).cpu().numpy())
    return out


def _suite_grad_finite_diff(seed: int) -> dict:
    """cli.py:250-285: 50 random small MLPs, analytic mlp_backward (device
    fp64) against central differences of the device forward, <= 1e-6."""
    import torch

    from . import tpnumerics as T
    if not torch.cuda.is_available():
        return _fail("grad-finite-diff", "needs a CUDA device (no CPU fallback)", {})
    rng = np.random.default_rng(seed)
    worst = 0.0
    for i in range(50):
        hidden = int(rng.integers(2, 6))
        ffn = int(rng.integers(3, 11))
        layer = T.MlpLayer.random(hidden, ffn, seed=int(rng.integers(2**31)))
        x = rng.standard_normal((3, hidden))
        g = rng.standard_normal((3, hidden))
        da, db = T.mlp_backward(x, layer, g)
        fd_a, fd_b = _central_differences(T, x, g, layer.A, layer.B)
        err = max(_rel_err(fd_a, da), _rel_err(fd_b, db))
        worst = max(worst, err)
        if err > 1e-6:
            return _fail("grad-finite-diff", "analytic gradient differs from central differences",
                         {"instance": i, "hidden": hidden, "ffn": ffn, "rel_err": err})
    return _ok("grad-finite-diff", f"50 instances, worst rel err {worst:.2e}")


def _golden_fixture() -> dict:
    """The reference's committed golden MLP fixture (configs/golden_mlp.json,
    h=4, ffn=16, seed 0), shipped with this package."""
    from importlib import resources
    return json.loads(resources.files(__package__).joinpath("configs/golden_mlp.json").read_text())


def _suite_golden(seed: int) -> dict:
    """cli.py:288-309: the seeded layer stream reproduces the fixture's A, B;
    the device forward and backward reproduce its Y, dA, dB within 1e-12."""
    import torch

    from . import tpnumerics as T
    del seed  # the fixture is fixed
    if not torch.cuda.is_available():
        return _fail("golden", "needs a CUDA device (no CPU fallback)", {})
    fx = _golden_fixture()
    layer = T.MlpLayer(A=np.array(fx["A"]), B=np.array(fx["B"]))
    regen = T.MlpLayer.random(fx["hidden"], fx["ffn"], seed=fx["seed"])
    if not (np.array_equal(regen.A, layer.A) and np.array_equal(regen.B, layer.B)):
        return _fail("golden", "seeded layer generation drifted from the fixture", {})
    x, g = np.array(fx["X"]), np.array(fx["G"])
    da, db = T.mlp_backward(x, layer, g)
    got = {"Y": T.mlp_forward_dense(x, layer), "dA": da, "dB": db}
    for name in ("Y", "dA", "dB"):
        err = _rel_err(got[name], np.array(fx[name]))
        if err > 1e-12:
            return _fail("golden", f"recomputed {name} differs from the committed fixture",
                         {"field": name, "rel_err": err})
    return _ok("golden", "forward and gradients match the committed fixture")


SUITES = {"shard-invariants": _suite_shard_invariants, "tp-numerics": _suite_tp_numerics,
          "grad-finite-diff": _suite_grad_finite_diff, "golden": _suite_golden}


def cmd_verify(args) -> int:
    names = list(SUITES) if args.suite == "all" else [args.suite]
    results = [SUITES[n](args.seed) for n in names]
    if args.json:
        print(json.dumps({"passed": all(r["passed"] for r in results), "suites": results}, indent=2))
    else:
        for r in results:
            print(f"{'PASS' if r['passed'] else 'FAIL'} {r['name']}: {r['detail']}")
            if r["case"]:
                print(f"     case: {json.dumps(r['case'])}")
    return 0 if all(r["passed"] for r in results) else 1


def _plan_stats(plan) -> dict:
    """cli.py:346-353."""
    return {"direction": plan.direction, "total_cols_moved": plan.total_cols_moved,
            "max_cols_sent": plan.max_cols_sent, "max_cols_received": plan.max_cols_received,
            "links": len(plan.transfers)}


def cmd_shardmap(args) -> int:
    """cli.py:356-382: same text lines and JSON document."""
    smap = build_shard_map(args.k, args.n1, args.n2)
    pre = build_reshard_plan(smap, PRE_SYNC)
    post = build_reshard_plan(smap, POST_SYNC)
    if args.json:
        print(json.dumps({"map": smap.to_json_dict(), "pre_sync": _plan_stats(pre),
                          "post_sync": _plan_stats(post)}, indent=2))
        return 0
    comp, sync = smap.comp_counts(), smap.sync_counts()
    print(f"shard map: k={args.k} n1={args.n1} n2={args.n2}")
    print(f"  comp shards per rank: {comp.min()}..{comp.max()}")
    print(f"  sync shards per rank: {sync.min()}..{sync.max()} on {args.n2} ranks")
    for name, plan in (("pre-sync", pre), ("post-sync", post)):
        print(f"  {name}: {plan.total_cols_moved} columns over {len(plan.transfers)} links, "
              f"max {plan.max_cols_sent} sent / {plan.max_cols_received} received per rank")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="ntp-b200", description="NTP shard maps and B200 sync verification")
    ap.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("shardmap", help="print a shard map and reshard-plan statistics")
    p.add_argument("--k", type=int, required=True)
    p.add_argument("--n1", type=int, required=True)
    p.add_argument("--n2", type=int, required=True)
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_shardmap)
    p = sub.add_parser("verify", help="run the oracle suites against this implementation")
    p.add_argument("--suite", choices=["all", *SUITES], default="all")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_verify)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError, json.JSONDecodeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
