"""Fused weight-gradient GEMM + NTP sync (ntp_gemm_bf16_red): every replica's
tcgen05 wgrad epilogue red.adds its batch-weighted gradient into its own
unit-major arena and the partner replica's.  Checked against the unfused path
(tcgen05 wgrad -> nonuniform_grad_sync) and against the fp64 oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import linear, tpnumerics
    return linear, tpnumerics


@pytest.mark.parametrize("mode", ["red", "red_tma"])
@pytest.mark.parametrize("gdtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 1e-2)])
def test_fused_backward_sync_matches_unfused(mods, gdtype, tol, mode):
    """mode "red": per-thread red.add; "red_tma": TMA bulk tensor reductions of
    whole 32 x 32 boxes into both arenas (row red.adds at run boundaries)."""
    Lin, T = mods
    from paper_2504_06095_b200.shardmap import build_shard_map
    h, k, tok_h, tok_r = 128, 1000, 256, 192
    A, B = O.random_layer(h, k, seed=11)
    A, B = A / np.sqrt(h), B / np.sqrt(k)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    r64 = lambda x: bf(x).double().numpy()  # noqa: E731
    A, B = r64(A), r64(B)
    rng = np.random.default_rng(12)
    Xh, Gh = (r64(rng.standard_normal((tok_h, h))) for _ in range(2))
    Xr, Gr = (r64(rng.standard_normal((tok_r, h))) for _ in range(2))
    smap = build_shard_map(k, 4, 3)
    hc, rc = T.assignment_from_comp(smap), T.assignment_from_sync(smap)
    w_h, w_r = tok_h / (tok_h + tok_r), tok_r / (tok_h + tok_r)
    layer = T.MlpLayer(A, B)
    sh_h = [Lin.MlpShard(A, B, c) for c in hc]
    sh_r = [Lin.MlpShard(A, B, c) for c in rc]
    for sh in sh_h:
        sh.forward(bf(Xh).cuda(), torch.empty((tok_h, h), device="cuda"))
    for sh in sh_r:
        sh.forward(bf(Xr).cuda(), torch.empty((tok_r, h), device="cuda"))
    # unfused: wgrad -> nonuniform_grad_sync
    uh = T.MlpReplica(layer, hc, dtype=gdtype)
    ur = T.MlpReplica(layer, rc, dtype=gdtype)
    Lin.mlp_backward_tp(bf(Xh).cuda(), sh_h, bf(Gh).cuda(), uh)
    Lin.mlp_backward_tp(bf(Xr).cuda(), sh_r, bf(Gr).cuda(), ur)
    T.nonuniform_grad_sync(uh, ur, smap, weights=(w_h, w_r))
    # fused: both replicas push into zeroed arenas
    fh = T.MlpReplica(layer, hc, dtype=gdtype)
    fr = T.MlpReplica(layer, rc, dtype=gdtype)
    for sh, cols, g in zip(sh_h, hc, fh.grads):
        rb, rr = Lin.partner_row_map(cols, rc, "cuda")
        sh.backward_synced(bf(Xh).cuda(), bf(Gh).cuda(), g, w_h, rb, rr, fr.grads, mode=mode)
    for sh, cols, g in zip(sh_r, rc, fr.grads):
        rb, rr = Lin.partner_row_map(cols, hc, "cuda")
        sh.backward_synced(bf(Xr).cuda(), bf(Gr).cuda(), g, w_r, rb, rr, fh.grads, mode=mode)
    fh._has_grads = fr._has_grads = True
    torch.cuda.synchronize()
    # both replicas identical bit for bit
    dh, dr = fh.dense_grads(), fr.dense_grads()
    assert np.array_equal(dh[0], dr[0]) and np.array_equal(dh[1], dr[1])
    uh_d = uh.dense_grads()
    for got, want in zip(dh, uh_d):
        assert O.rel_err(got, want) < tol
    # and against the fp64 oracle of the weighted dense sum
    da1, db1 = O.mlp_backward(Xh, A, B, Gh)
    da2, db2 = O.mlp_backward(Xr, A, B, Gr)
    assert O.rel_err(dh[0], w_h * da1 + w_r * da2) < 2e-2
    assert O.rel_err(dh[1], w_h * db1 + w_r * db2) < 2e-2


@pytest.mark.parametrize("mode", ["push", "push_tma"])
@pytest.mark.parametrize("gdtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 1e-2)])
def test_fused_push_mode(mods, gdtype, tol, mode):
    """mode "push": plain stores into the partner's staging arena, then each
    replica adds its staging locally -- same result, replicas bit-identical.
    "push_tma": 32-row boxes that are consecutive in the partner's layout go as
    TMA tensor stores, the rest (run boundaries, ragged tails) as row stores."""
    Lin, T = mods
    from paper_2504_06095_b200.shardmap import build_shard_map
    h, k, tok_h, tok_r = 128, 600, 256, 192
    A, B = O.random_layer(h, k, seed=21)
    A, B = A / np.sqrt(h), B / np.sqrt(k)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    r64 = lambda x: bf(x).double().numpy()  # noqa: E731
    A, B = r64(A), r64(B)
    rng = np.random.default_rng(22)
    Xh, Gh = (r64(rng.standard_normal((tok_h, h))) for _ in range(2))
    Xr, Gr = (r64(rng.standard_normal((tok_r, h))) for _ in range(2))
    smap = build_shard_map(k, 4, 3)
    hc, rc = T.assignment_from_comp(smap), T.assignment_from_sync(smap)
    w_h, w_r = tok_h / (tok_h + tok_r), tok_r / (tok_h + tok_r)
    layer = T.MlpLayer(A, B)
    sh_h = [Lin.MlpShard(A, B, c) for c in hc]
    sh_r = [Lin.MlpShard(A, B, c) for c in rc]
    for sh in sh_h:
        sh.forward(bf(Xh).cuda(), torch.empty((tok_h, h), device="cuda"))
    for sh in sh_r:
        sh.forward(bf(Xr).cuda(), torch.empty((tok_r, h), device="cuda"))
    fh, fr = T.MlpReplica(layer, hc, dtype=gdtype), T.MlpReplica(layer, rc, dtype=gdtype)
    sth, stf = T.MlpReplica(layer, hc, dtype=gdtype), T.MlpReplica(layer, rc, dtype=gdtype)
    for sh, cols, g in zip(sh_h, hc, fh.grads):
        rb, rr = Lin.partner_row_map(cols, rc, "cuda")
        sh.backward_synced(bf(Xh).cuda(), bf(Gh).cuda(), g, w_h, rb, rr, stf.grads, mode=mode)
    for sh, cols, g in zip(sh_r, rc, fr.grads):
        rb, rr = Lin.partner_row_map(cols, hc, "cuda")
        sh.backward_synced(bf(Xr).cuda(), bf(Gr).cuda(), g, w_r, rb, rr, sth.grads, mode=mode)
    for g, s in zip(fh.grads + fr.grads, sth.grads + stf.grads):
        Lin.finish_push(g, s)
    fh._has_grads = fr._has_grads = True
    torch.cuda.synchronize()
    dh, dr = fh.dense_grads(), fr.dense_grads()
    assert np.array_equal(dh[0], dr[0]) and np.array_equal(dh[1], dr[1])
    da1, db1 = O.mlp_backward(Xh, A, B, Gh)
    da2, db2 = O.mlp_backward(Xr, A, B, Gr)
    assert O.rel_err(dh[0], w_h * da1 + w_r * da2) < 2e-2
    assert O.rel_err(dh[1], w_h * db1 + w_r * db2) < 2e-2
