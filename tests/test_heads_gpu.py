"""Attention heads as sync units (the reference shards attention by heads,
tpnumerics.py:158-217, but has no attention gradients): head units of
4*hidden*head_dim elements through the same kernel, vs the oracle."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("heads,n1,n2,dtype,tol", [(32, 4, 3, torch.bfloat16, 2e-2),
                                                   (16, 4, 3, torch.float32, 1e-6),
                                                   (128, 32, 30, torch.bfloat16, 2e-2),
                                                   (7, 2, 1, torch.float32, 1e-6)])
def test_head_sync_vs_oracle(heads, n1, n2, dtype, tol):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import tpnumerics as T
    from paper_2504_06095_b200.shardmap import attention_head_partition, build_shard_map
    layer = SimpleNamespace(heads=heads, hidden=64, head_dim=16)
    smap = build_shard_map(heads, n1, n2)
    counts, _ = attention_head_partition(heads, n2)
    assert smap.sync_counts().tolist() == counts.tolist()
    hc, rc = T.assignment_from_comp(smap), T.assignment_from_sync(smap)
    unit = 4 * 64 * 16
    rng = np.random.default_rng(heads)
    rnd = lambda a: torch.from_numpy(a).to(dtype).double().numpy()  # noqa: E731
    hu = [rnd(rng.standard_normal((len(c), unit))) for c in hc]
    ru = [rnd(rng.standard_normal((len(c), unit))) for c in rc]
    h = T.AttentionReplica(layer, hc, dtype=dtype).set_units(hu)
    r = T.AttentionReplica(layer, rc, dtype=dtype).set_units(ru)
    T.nonuniform_head_sync(h, r, smap, weights=(0.6, 0.4))
    hb = [u.ravel().copy() for u in hu]
    rb = [u.ravel().copy() for u in ru]
    O.nonuniform_sync(smap.comp_rank, smap.sync_rank, hc, rc, hb, rb, unit,
                      op=O.OP_WEIGHTED, weights=(0.6, 0.4))
    for rep, want in ((h, hb), (r, rb)):
        got = np.concatenate([u.ravel() for u in rep.units()])
        assert O.rel_err(got, np.concatenate(want)) <= tol
    with pytest.raises(ValueError, match="map is over k="):
        T.nonuniform_head_sync(h, r, build_shard_map(heads + 1, n1, n2))
