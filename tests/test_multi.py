"""DP > 2 sync across replicas of mixed layouts (BASELINE configs[2]: DP=4 x TP2
with one replica degraded to TP1, batch-proportional weights).

No reference function exists for R > 2 nonuniform replicas, so the oracle is
the reference's uniform_grad_sync arithmetic (tpnumerics.py:263-286, restated
in oracle.uniform_sync) applied to the replicas' dense (column-ordered)
gradients: per-unit arithmetic does not depend on where a unit is stored."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2504_06095_b200.plans import MultiPlan

from test_sync_gpu import _round


def test_multiplan_host_checks():
    p = MultiPlan(1, 4)
    p.add_units(8, np.zeros((4, 3), dtype=np.int32) + np.arange(4)[:, None],
                np.arange(3)[None, :] * 8 + np.zeros((4, 1), dtype=np.int64)).finalize()
    assert p.n_chunks == 1  # three contiguous units merge into one run
    with pytest.raises(ValueError):
        MultiPlan(1, 9)
    with pytest.raises(ValueError):
        MultiPlan(1, 2).add_units(8, [[0]], [[0]])
    q = MultiPlan(0, 2).add_units(3, [[0], [1]], [[0], [0]])
    with pytest.raises(ValueError, match="16-byte"):
        q.finalize()


def _layouts(k):
    from paper_2504_06095_b200 import tpnumerics as T
    from paper_2504_06095_b200.shardmap import build_shard_map
    tp2 = T.assignment_from_comp(build_shard_map(k, 2, 1))
    tp1 = T.assignment_from_sync(build_shard_map(k, 2, 1))
    m43 = build_shard_map(k, 4, 3)
    return tp2, tp1, T.assignment_from_comp(m43), T.assignment_from_sync(m43)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [1, 2], ids=["ldg", "bulk"])
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-6), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("mode", ["c3", "mixed"])
def test_multi_sync_vs_oracle(dtype, tol, mode, variant):
    """Both kernels (128-bit loads; TMA-bulk ring, R <= 4 -- "mixed" has R = 5
    and keeps the load kernel) against the oracle, and bit-identical to each
    other (the same explicitly rounded arithmetic in the same order)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import _lib
    _lib.load().ntp_multi_set_kernel(variant)
    try:
        _multi_case(dtype, tol, mode)
    finally:
        _lib.load().ntp_multi_set_kernel(0)


_RESULTS = {}


def _multi_case(dtype, tol, mode):
    from paper_2504_06095_b200 import tpnumerics as T
    k, h = 2000, 32
    tp2, tp1, comp43, sync43 = _layouts(k)
    if mode == "c3":   # DP=4 x TP2, one replica degraded to TP1; TP1 has half the local batch
        layouts, w = [tp2, tp2, tp2, tp1], np.array([2, 2, 2, 1]) / 7
    else:              # TP4 (NTP comp), TP4, TP3, TP2, TP1 together
        layouts, w = [comp43, comp43, sync43, tp2, tp1], np.array([4, 4, 3, 2, 1]) / 14
    layer = T.MlpLayer(np.zeros((h, k)), np.zeros((k, h)))
    rng = np.random.default_rng(0)
    dense = [_round(rng.standard_normal((k, 2 * h)), dtype) for _ in layouts]
    reps = [T.MlpReplica(layer, cols, dtype=dtype).set_units([d[c] for c in cols])
            for cols, d in zip(layouts, dense)]
    for op, weights, code in (("sum", w, O.OP_WEIGHTED), ("sum", None, O.OP_SUM),
                              ("mean", None, O.OP_MEAN)):
        for rep, cols, d in zip(reps, layouts, dense):
            rep.set_units([d[c] for c in cols])
        T.multi_grad_sync(reps, op=op, weights=weights)
        want = [d.ravel().copy() for d in dense]
        O.uniform_sync(want, op=code, weights=weights)
        want = want[0].reshape(k, 2 * h)
        first = None
        for rep, cols in zip(reps, layouts):
            got = np.zeros((k, 2 * h))
            for c, u in zip(cols, rep.units()):
                got[c] = u
            assert O.rel_err(got, want) <= tol, (op, O.rel_err(got, want))
            first = got if first is None else first
            assert np.array_equal(got, first)  # every replica holds identical bits
        key = (str(dtype), mode, op, code)
        if key in _RESULTS:  # the other kernel variant ran first: same bits
            assert np.array_equal(_RESULTS[key], first)
        _RESULTS[key] = first


@pytest.mark.gpu
def test_multi_sync_validation():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import tpnumerics as T
    layer = T.MlpLayer(np.zeros((4, 16)), np.zeros((16, 4)))
    a = T.MlpReplica(layer, T.contiguous_assignment(16, 2))
    b = T.MlpReplica(layer, T.contiguous_assignment(16, 1))
    with pytest.raises(ValueError, match="holds no gradients"):
        T.multi_grad_sync([a, b])
    a.set_units([np.zeros((8, 8))] * 2)
    b.set_units([np.zeros((16, 8))])
    with pytest.raises(ValueError, match="unknown reduction op"):
        T.multi_grad_sync([a, b], op="max")
    with pytest.raises(ValueError, match="one weight per replica"):
        T.multi_grad_sync([a, b], weights=[1.0])
