"""Drop-in check: the reference's tpnumerics call sites against this package.

Each test drives ``paper_2504_06095_b200.tpnumerics`` exactly as the
reference's own tests drive ``ntpsim.tpnumerics`` (pkg/tests/test_tpnumerics.py,
same names, argument order, default dtypes and 1e-12 tolerances) -- only the
import differs -- plus the bf16 dispatch of ``mlp_backward_tp`` /
``mlp_forward_tp`` onto the tcgen05 GEMMs and the numpy-object host path.
"""

import json

import numpy as np
import pytest
import torch

from oracle import oracle as O

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
RTOL = 1e-12


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import tpnumerics
    return tpnumerics


@pytest.fixture(scope="module")
def smaps():
    from paper_2504_06095_b200.shardmap import build_shard_map
    return build_shard_map


def rel(got, want):
    return O.rel_err(np.asarray(got), np.asarray(want))


def _cases(n, seed=0):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        n1 = int(rng.integers(2, 13))
        n2 = int(rng.integers(1, n1 + 1))
        k = int(rng.integers(n1, 97))
        yield k, n1, n2, int(rng.integers(2, 6)), int(rng.integers(0, 2**20))


def test_forward_tp_matches_dense_on_both_layouts(T, smaps):
    for k, n1, n2, hidden, seed in _cases(30):
        rng = np.random.default_rng(seed)
        layer = T.MlpLayer.random(hidden, k, seed=seed)
        smap = smaps(k, n1, n2)
        x = rng.standard_normal((3, hidden))
        want = T.mlp_forward_dense(x, layer)
        assert isinstance(want, np.ndarray) and want.shape == (3, hidden)
        for assignment in (T.assignment_from_comp(smap), T.assignment_from_sync(smap)):
            rep = T.MlpReplica(layer, assignment)
            assert rel(T.mlp_forward_tp(x, rep), want) < RTOL
            assert all(np.array_equal(a, layer.A[:, c]) for a, c in zip(rep.a_frags, rep.cols))
            assert all(np.array_equal(b, layer.B[c, :]) for b, c in zip(rep.b_frags, rep.cols))


def test_nonuniform_sync_equals_dense_sum_default_dtype(T, smaps):
    for k, n1, n2, hidden, seed in _cases(30, seed=1):
        rng = np.random.default_rng(seed)
        layer = T.MlpLayer.random(hidden, k, seed=seed)
        smap = smaps(k, n1, n2)
        healthy = T.MlpReplica(layer, T.assignment_from_comp(smap))
        reduced = T.MlpReplica(layer, T.assignment_from_sync(smap))
        x1, x2 = rng.standard_normal((2, 4, hidden))
        g1, g2 = rng.standard_normal((2, 4, hidden))
        T.mlp_backward_tp(x1, healthy, g1)
        T.mlp_backward_tp(x2, reduced, g2)
        T.nonuniform_grad_sync(healthy, reduced, smap)
        da1, db1 = T.mlp_backward(x1, layer, g1)
        da2, db2 = T.mlp_backward(x2, layer, g2)
        for rep in (healthy, reduced):
            da, db = rep.dense_grads()
            assert rel(da, da1 + da2) < RTOL and rel(db, db1 + db2) < RTOL


def test_mlp_backward_matches_oracle(T):
    rng = np.random.default_rng(4)
    A, B = O.random_layer(5, 12, seed=4)
    x, g = rng.standard_normal((2, 3, 5))
    da, db = T.mlp_backward(x, T.MlpLayer(A, B), g)
    wa, wb = O.mlp_backward(x, A, B, g)
    assert rel(da, wa) < RTOL and rel(db, wb) < RTOL
    with pytest.raises(ValueError, match="upstream grad shape"):
        T.mlp_backward(x, T.MlpLayer(A, B), g[:, :4])
    with pytest.raises(ValueError, match="X has 4 features, layer expects 5"):
        T.mlp_forward_dense(x[:, :4], T.MlpLayer(A, B))


def test_gelu_grad_matches_finite_differences(T):
    x = np.linspace(-4, 4, 41)
    h = 1e-7
    fd = (T.gelu(x + h) - T.gelu(x - h)) / (2 * h)
    assert np.max(np.abs(fd - T.gelu_grad(x))) < 1e-6
    assert rel(T.gelu(x), O.gelu(x)) < RTOL  # device vs numpy tanh: ulp-level


def test_attention_tp_matches_dense(T):
    rng = np.random.default_rng(11)
    for _ in range(20):
        heads = int(rng.integers(2, 9))
        head_dim = int(rng.integers(2, 5))
        hidden = int(rng.integers(3, 7))
        n = int(rng.integers(1, heads + 1))
        layer = T.AttentionLayer.random(heads, hidden, head_dim, seed=int(rng.integers(2**31)))
        rep = T.AttentionReplica(layer, T.contiguous_assignment(heads, n))
        x = rng.standard_normal((5, hidden))
        assert rel(T.attention_forward_tp(x, rep), T.attention_forward_dense(x, layer)) < RTOL


def test_golden_fixture_reproduced(T):
    with open(f"{GOLDEN}/golden_mlp.json") as f:
        fx = json.load(f)
    layer = T.MlpLayer(np.array(fx["A"]), np.array(fx["B"]))
    x, g = np.array(fx["X"]), np.array(fx["G"])
    assert rel(T.mlp_forward_dense(x, layer), np.array(fx["Y"])) < RTOL
    da, db = T.mlp_backward(x, layer, g)
    assert rel(da, np.array(fx["dA"])) < RTOL and rel(db, np.array(fx["dB"])) < RTOL


def test_golden_detects_activation_drift(T, monkeypatch):
    with open(f"{GOLDEN}/golden_mlp.json") as f:
        fx = json.load(f)
    layer = T.MlpLayer(np.array(fx["A"]), np.array(fx["B"]))
    monkeypatch.setattr(T, "GELU_C", 0.0447)
    assert rel(T.mlp_forward_dense(np.array(fx["X"]), layer), np.array(fx["Y"])) > RTOL


def test_bf16_replica_backward_runs_tcgen05(T, smaps):
    """bf16 replicas: mlp_backward_tp / mlp_forward_tp dispatch to the tcgen05
    GEMMs (linear.MlpShard); gradients and forward within 2e-2 of fp64."""
    from paper_2504_06095_b200 import linear
    rng = np.random.default_rng(7)
    hidden, k = 128, 600
    A, B = O.random_layer(hidden, k, seed=7)
    A, B = A / np.sqrt(hidden), B / np.sqrt(k)
    layer = T.MlpLayer(A, B)
    smap = smaps(k, 4, 3)
    x, g = rng.standard_normal((2, 256, hidden))
    calls = []
    orig, orig_red = linear.mm, linear.mm_red
    monkey = pytest.MonkeyPatch()
    monkey.setattr(linear, "mm", lambda *a, **kw: calls.append(1) or orig(*a, **kw))
    monkey.setattr(linear, "mm_red", lambda *a, **kw: calls.append(1) or orig_red(*a, **kw))
    try:
        for assignment in (T.assignment_from_comp(smap), T.assignment_from_sync(smap)):
            rep = T.MlpReplica(layer, assignment, dtype=torch.bfloat16)
            T.mlp_backward_tp(x, rep, g)
            ref = T.MlpReplica(layer, assignment)
            T.mlp_backward_tp(x, ref, g)
            for got, want in zip(rep.dense_grads(), ref.dense_grads()):
                assert rel(got, want) < 2e-2
            z = T.mlp_forward_tp(x, rep)
            assert rel(z, T.mlp_forward_dense(x, layer)) < 2e-2
    finally:
        monkey.undo()
    assert len(calls) >= 2 * (4 + 3) * 3


def test_numpy_objects_host_path_cached(T, smaps):
    """The reference's own numpy replicas go through pinned staging + the fp64
    kernel; the second call reuses the cached plan and buffers."""
    from types import SimpleNamespace
    k, hidden = 96, 6
    A, B = O.random_layer(hidden, k, seed=2)
    smap = smaps(k, 4, 3)
    rng = np.random.default_rng(2)
    hc, rc = T.assignment_from_comp(smap), T.assignment_from_sync(smap)

    def np_replica(cols, x, g):
        frags = O.mlp_backward_tp(x, A, B, g, cols)
        return SimpleNamespace(layer=T.MlpLayer(A, B), n=len(cols), cols=cols,
                               grad_a=[f[0] for f in frags], grad_b=[f[1] for f in frags])
    for it in range(2):
        x1, x2, g1, g2 = rng.standard_normal((4, 4, hidden))
        h, r = np_replica(hc, x1, g1), np_replica(rc, x2, g2)
        ids = [id(a) for a in h.grad_a + r.grad_a]
        T.nonuniform_grad_sync(h, r, smap)
        assert ids == [id(a) for a in h.grad_a + r.grad_a]  # mutated in place
        want_a, want_b = (a + b for a, b in zip(O.mlp_backward(x1, A, B, g1),
                                                O.mlp_backward(x2, A, B, g2)))
        for rep in (h, r):
            da, db = np.zeros((hidden, k)), np.zeros((k, hidden))
            for c, ga, gb in zip(rep.cols, rep.grad_a, rep.grad_b):
                da[:, c], db[c, :] = ga, gb
            assert rel(da, want_a) < RTOL and rel(db, want_b) < RTOL
    assert len(T._HOST_PATHS) >= 1
