"""Parity of the device gradient sync (libntp_b200.so) with the CPU oracle.

Inputs are produced by the oracle's restatement of the reference's gradient
producer (fp64), cast to the device dtype; the expected output is the
oracle's fp64 nonuniform_grad_sync run on the same (cast) values.  Tolerances
(north_star): fp32 <= 1e-6, bf16 <= 2e-2 Frobenius relative error; fp64 and
the reference's own outputs are compared bit for bit.
"""

import json
import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import oracle as O

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 0.0, torch.float32: 1e-6, torch.bfloat16: 2e-2, torch.float16: 2e-3}


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import tpnumerics
    return tpnumerics


def _round(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype).to(torch.float64).numpy()


def make_case(T, k, n1, n2, hidden, seed, dtype, batch=4, rng=None, permute=False):
    """Device replicas + fp64 oracle buffers holding the same (dtype-rounded) grads."""
    from paper_2504_06095_b200.shardmap import build_shard_map
    rng = np.random.default_rng(seed) if rng is None else rng
    A, B = O.random_layer(hidden, k, seed=seed)
    smap = build_shard_map(k, n1, n2)
    hc = T.assignment_from_comp(smap)
    rc = T.assignment_from_sync(smap)
    if permute:  # the reference accepts any column order inside a rank (tpnumerics.py:304-311)
        hc = [rng.permutation(c) for c in hc]
        rc = [rng.permutation(c) for c in rc]
    x1, x2 = rng.standard_normal((2, batch, hidden))
    g1, g2 = rng.standard_normal((2, batch, hidden))
    hu = [_round(O.to_units(*g), dtype) for g in O.mlp_backward_tp(x1, A, B, g1, hc)]
    ru = [_round(O.to_units(*g), dtype) for g in O.mlp_backward_tp(x2, A, B, g2, rc)]
    layer = T.MlpLayer(A, B)
    healthy = T.MlpReplica(layer, hc, dtype=dtype).set_units(hu)
    reduced = T.MlpReplica(layer, rc, dtype=dtype).set_units(ru)
    return smap, healthy, reduced, hu, ru


def oracle_sync(smap, healthy, reduced, hu, ru, op=O.OP_SUM, w=(1.0, 1.0)):
    hb = [np.ascontiguousarray(u.ravel()) for u in hu]
    rb = [np.ascontiguousarray(u.ravel()) for u in ru]
    O.nonuniform_sync(smap.comp_rank, smap.sync_rank, healthy.cols, reduced.cols, hb, rb,
                      2 * healthy.hidden, op=op, weights=w)
    return hb, rb


def check(rep, want_bufs, dtype):
    got = np.concatenate([u.ravel() for u in rep.units()])
    want = np.concatenate(want_bufs)
    if TOL[dtype] == 0.0:
        assert np.array_equal(got, want)
    else:
        err = O.rel_err(got, want)
        assert err <= TOL[dtype], err
    return got


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_crit01_hundred_instances(T, dtype):
    """Acceptance criterion 01's instance distribution (test_acceptance.py:67-97)."""
    rng = np.random.default_rng(0)
    for _ in range(100):
        n1 = int(rng.integers(2, 17))
        n2 = int(rng.integers(1, n1 + 1))
        k = int(rng.integers(n1, 513))
        hidden = int(rng.integers(2, 7))
        seed = int(rng.integers(2**31))
        smap, h, r, hu, ru = make_case(T, k, n1, n2, hidden, seed, dtype, rng=rng)
        T.nonuniform_grad_sync(h, r, smap)
        hb, rb = oracle_sync(smap, h, r, hu, ru)
        gh = check(h, hb, dtype)
        gr = check(r, rb, dtype)
        # both replicas end with identical bits (tpnumerics.py:346-347, 355-356)
        da_h, db_h = h.dense_grads()
        da_r, db_r = r.dense_grads()
        assert np.array_equal(da_h, da_r) and np.array_equal(db_h, db_r)
        del gh, gr


def test_reference_outputs_bit_exact_fp64(T):
    """The reference's own nonuniform_grad_sync outputs (tests/golden)."""
    meta = json.load(open(os.path.join(GOLDEN, "sync_cases.json")))["cases"]
    npz = np.load(os.path.join(GOLDEN, "sync_cases.npz"))
    from paper_2504_06095_b200.shardmap import build_shard_map
    for c in meta:
        smap = build_shard_map(c["k"], c["n1"], c["n2"])
        A, B = O.random_layer(c["hidden"], c["k"], seed=c["seed"])
        layer = T.MlpLayer(A, B)
        u = 2 * c["hidden"]
        h = T.MlpReplica(layer, T.assignment_from_comp(smap), dtype=torch.float64)
        r = T.MlpReplica(layer, T.assignment_from_sync(smap), dtype=torch.float64)
        h.set_units(np.split(npz[c["tag"] + "_h_in"], np.cumsum(c["h_counts"])[:-1] * u))
        r.set_units(np.split(npz[c["tag"] + "_r_in"], np.cumsum(c["r_counts"])[:-1] * u))
        T.nonuniform_grad_sync(h, r, smap, op=c["op"])
        assert np.array_equal(np.concatenate([x.ravel() for x in h.units()]), npz[c["tag"] + "_h_out"])
        assert np.array_equal(np.concatenate([x.ravel() for x in r.units()]), npz[c["tag"] + "_r_out"])


def test_reference_objects_host_path(T):
    """Reference-shaped numpy replicas go host->device->host, bit-exact fp64."""
    meta = json.load(open(os.path.join(GOLDEN, "sync_cases.json")))["cases"]
    npz = np.load(os.path.join(GOLDEN, "sync_cases.npz"))
    from paper_2504_06095_b200.shardmap import build_shard_map
    for c in meta[:8]:
        smap = build_shard_map(c["k"], c["n1"], c["n2"])
        A, B = O.random_layer(c["hidden"], c["k"], seed=c["seed"])
        layer = SimpleNamespace(A=A, B=B, hidden=c["hidden"], ffn=c["k"])
        hid, u = c["hidden"], 2 * c["hidden"]

        def rep(cols, flat, counts):
            parts = np.split(flat, np.cumsum(counts)[:-1] * u)
            ga = [O.from_units(p, hid)[0] for p in parts]
            gb = [O.from_units(p, hid)[1] for p in parts]
            return SimpleNamespace(layer=layer, n=len(cols), cols=cols, grad_a=ga, grad_b=gb)

        h = rep(T.assignment_from_comp(smap), npz[c["tag"] + "_h_in"], c["h_counts"])
        r = rep(T.assignment_from_sync(smap), npz[c["tag"] + "_r_in"], c["r_counts"])
        ga0 = h.grad_a[0]
        T.nonuniform_grad_sync(h, r, smap, op=c["op"])
        assert h.grad_a[0] is ga0  # mutated in place, like the reference
        got = np.concatenate([O.to_units(a, b).ravel() for a, b in zip(h.grad_a, h.grad_b)])
        assert np.array_equal(got, npz[c["tag"] + "_h_out"])
        got = np.concatenate([O.to_units(a, b).ravel() for a, b in zip(r.grad_a, r.grad_b)])
        assert np.array_equal(got, npz[c["tag"] + "_r_out"])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
def test_weighting(T, dtype):
    smap, h, r, hu, ru = make_case(T, 300, 8, 5, 16, 7, dtype)
    T.nonuniform_grad_sync(h, r, smap, weights=(4 / 7, 3 / 7))
    hb, rb = oracle_sync(smap, h, r, hu, ru, op=O.OP_WEIGHTED, w=(4 / 7, 3 / 7))
    check(h, hb, dtype)
    check(r, rb, dtype)
    # (1, 1) is op "sum" and (1/2, 1/2) is op "mean", bit for bit
    for w, op in (((1.0, 1.0), "sum"), ((0.5, 0.5), "mean")):
        s1, h1, r1, _, _ = make_case(T, 300, 8, 5, 16, 7, dtype)
        s2, h2, r2, _, _ = make_case(T, 300, 8, 5, 16, 7, dtype)
        T.nonuniform_grad_sync(h1, r1, s1, weights=w)
        T.nonuniform_grad_sync(h2, r2, s2, op=op)
        for a, b in zip(h1.units() + r1.units(), h2.units() + r2.units()):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_c1_config(T, dtype):
    """C1: h1024, ffn4096, TP4/TP3 with the SURVEY 8(d) inputs (rng 0, batches 4 and 3)."""
    from paper_2504_06095_b200.shardmap import build_shard_map
    A, B = O.random_layer(1024, 4096, seed=0)
    smap = build_shard_map(4096, 4, 3)
    rng = np.random.default_rng(0)
    xh, gh = rng.standard_normal((4, 1024)), rng.standard_normal((4, 1024))
    xr, gr = rng.standard_normal((3, 1024)), rng.standard_normal((3, 1024))
    hc, rc = T.assignment_from_comp(smap), T.assignment_from_sync(smap)
    hu = [_round(O.to_units(*g), dtype) for g in O.mlp_backward_tp(xh, A, B, gh, hc)]
    ru = [_round(O.to_units(*g), dtype) for g in O.mlp_backward_tp(xr, A, B, gr, rc)]
    layer = T.MlpLayer(A, B)
    h = T.MlpReplica(layer, hc, dtype=dtype).set_units(hu)
    r = T.MlpReplica(layer, rc, dtype=dtype).set_units(ru)
    T.nonuniform_grad_sync(h, r, smap, weights=(4 / 7, 3 / 7))
    hb, rb = oracle_sync(smap, h, r, hu, ru, op=O.OP_WEIGHTED, w=(4 / 7, 3 / 7))
    check(h, hb, dtype)
    check(r, rb, dtype)


@pytest.mark.parametrize("k,n1,n2,hidden", [(96, 8, 8, 4), (37, 16, 1, 3), (16, 16, 15, 8),
                                            (513, 16, 9, 5), (4, 4, 1, 2), (1, 1, 1, 2)])
def test_edge_cases(T, k, n1, n2, hidden):
    """n1 == n2 (aligned), n2 == 1, k == n1, ragged remainders, misaligned units."""
    for dtype in (torch.float64, torch.float32):
        smap, h, r, hu, ru = make_case(T, k, n1, n2, hidden, k + n1, dtype)
        T.nonuniform_grad_sync(h, r, smap, op="mean")
        hb, rb = oracle_sync(smap, h, r, hu, ru, op=O.OP_MEAN)
        check(h, hb, dtype)
        check(r, rb, dtype)


def test_permuted_rank_layouts(T):
    smap, h, r, hu, ru = make_case(T, 200, 6, 4, 8, 3, torch.float64, permute=True)
    T.nonuniform_grad_sync(h, r, smap)
    hb, rb = oracle_sync(smap, h, r, hu, ru)
    check(h, hb, torch.float64)
    check(r, rb, torch.float64)


def test_uniform_sync_reference_outputs(T):
    npz = np.load(os.path.join(GOLDEN, "sync_cases.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "sync_cases.json")))["uniform"]
    counts = npz["u_counts"]
    assignment = np.split(npz["u_cols"], np.cumsum(counts)[:-1])
    A, B = O.random_layer(meta["hidden"], meta["k"], seed=meta["layer_seed"])
    u = 2 * meta["hidden"]
    for op in ("sum", "mean"):
        reps = []
        for flat in npz[f"u_{op}_in"]:
            rep = T.MlpReplica(T.MlpLayer(A, B), assignment, dtype=torch.float64)
            reps.append(rep.set_units(np.split(flat, np.cumsum(counts)[:-1] * u)))
        T.uniform_grad_sync(reps, op=op)
        for rep, want in zip(reps, npz[f"u_{op}_out"]):
            assert np.array_equal(np.concatenate([x.ravel() for x in rep.units()]), want)


def test_validation_messages(T):
    smap, h, r, _, _ = make_case(T, 24, 4, 3, 4, 0, torch.float32)
    from paper_2504_06095_b200.shardmap import build_shard_map
    with pytest.raises(ValueError, match=r"replica degrees \(3, 4\) do not match map \(4, 3\)"):
        T.nonuniform_grad_sync(r, h, smap)
    with pytest.raises(ValueError, match="map is over k=25 columns, layer has ffn=24"):
        T.nonuniform_grad_sync(h, r, build_shard_map(25, 4, 3))
    with pytest.raises(ValueError, match="unknown reduction op 'max'"):
        T.nonuniform_grad_sync(h, r, smap, op="max")
    bare = T.MlpReplica(h.layer, r.cols)
    with pytest.raises(ValueError, match="both replicas must hold gradients"):
        T.nonuniform_grad_sync(h, bare, smap)
    with pytest.raises(ValueError, match="healthy replica is not sharded"):
        T.nonuniform_grad_sync(T.MlpReplica(h.layer, T.contiguous_assignment(24, 4)), r, smap)
    with pytest.raises(ValueError, match="replicas are not identically sharded"):
        T.uniform_grad_sync([h, T.MlpReplica(h.layer, T.contiguous_assignment(24, 4))])


def test_full_size_bf16_layer_property(T):
    """C4-shaped MLP layer (h4096, ffn14336, TP4/TP3, bf16, 117 M elements per
    replica): size-independent properties -- both replicas bitwise identical,
    and equal to a torch fp32 evaluation of w_h*g_h + w_r*g_r per column."""
    from paper_2504_06095_b200.shardmap import build_shard_map
    k, h = 14336, 4096
    smap = build_shard_map(k, 4, 3)
    layer = SimpleNamespace(hidden=h, ffn=k)
    hc, rc = T.assignment_from_comp(smap), T.assignment_from_sync(smap)
    g = torch.Generator(device="cuda").manual_seed(0)
    healthy = _blank(T, layer, hc, g)
    reduced = _blank(T, layer, rc, g)
    dense_h = _dense(healthy, k)
    dense_r = _dense(reduced, k)
    want = (dense_h.float() * (4 / 7) + dense_r.float() * (3 / 7))
    T.nonuniform_grad_sync(healthy, reduced, smap, weights=(4 / 7, 3 / 7))
    got_h = _dense(healthy, k)
    got_r = _dense(reduced, k)
    assert torch.equal(got_h, got_r)
    err = ((got_h.float() - want).norm() / want.norm()).item()
    assert err <= 2e-2, err
    # fp32 FMA then one rounding: within half a bf16 ulp of the fp32 value
    assert ((got_h.float() - want).abs() <= want.abs() * 2**-8 + 1e-30).all()


def _blank(T, layer, cols, gen):
    rep = T.MlpReplica(layer, cols, dtype=torch.bfloat16)
    return rep.set_units([torch.randn((len(c), 2, layer.hidden), generator=gen, device="cuda")
                          for c in cols])


def _dense(rep, k):
    out = torch.empty((k, 2, rep.layer.hidden), dtype=rep.dtype, device="cuda")
    for g, c in zip(rep.grads, rep.cols):
        out[torch.as_tensor(c, device="cuda")] = g
    return out


@pytest.mark.parametrize("variant", [2, 3])
def test_bulk_kernel_variants_match_oracle(T, variant):
    """The TMA bulk-copy kernels give the same bits as the LDG kernel and meet
    the oracle tolerance (crit-01 subset + C1-sized case)."""
    from paper_2504_06095_b200 import _lib
    L = _lib.load()
    try:
        rng = np.random.default_rng(1)
        for i in range(30):
            n1 = int(rng.integers(2, 17))
            n2 = int(rng.integers(1, n1 + 1))
            k = int(rng.integers(n1, 513))
            hidden = int(rng.choice([4, 8, 64, 1024]))
            for dtype in (torch.float32, torch.bfloat16):
                _lib.check(L.ntp_set_option(0, 1))  # LDG reference variant
                s1, h1, r1, hu, ru = make_case(T, k, n1, n2, hidden, i, dtype)
                T.nonuniform_grad_sync(h1, r1, s1, weights=(0.25, 0.75))
                _lib.check(L.ntp_set_option(0, variant))
                s2, h2, r2, _, _ = make_case(T, k, n1, n2, hidden, i, dtype)
                T.nonuniform_grad_sync(h2, r2, s2, weights=(0.25, 0.75))
                for a, b in zip(h1.units() + r1.units(), h2.units() + r2.units()):
                    assert np.array_equal(a, b)
                hb, rb = oracle_sync(s2, h2, r2, hu, ru, op=O.OP_WEIGHTED, w=(0.25, 0.75))
                check(h2, hb, dtype)
                check(r2, rb, dtype)
    finally:
        _lib.check(L.ntp_set_option(0, 0))  # back to AUTO
