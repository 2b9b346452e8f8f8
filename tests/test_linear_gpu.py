"""tcgen05 uneven-shard linears (ntp_gemm_bf16 / paper_2504_06095_b200.linear).

Floating-point kernel: each GEMM is checked against a plain torch fp32
evaluation of the same bf16 operands; the TP MLP chain against the oracle's
fp64 restatement of the reference (mlp_backward_tp, tpnumerics.py:238-252)
with the bf16 tolerance of the north_star (2e-2 Frobenius)."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[3, 2, 4, 0], ids=["pair256", "pair128", "pair224", "single"])
def Lin(request):
    """Both tile paths: CTA pairs (tcgen05 cta_group::2) and single CTAs."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import _lib, linear
    _lib.load().ntp_gemm_set_pair(request.param)  # 1 auto (pair tiles), 0 single-CTA
    yield linear
    _lib.load().ntp_gemm_set_pair(1)


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def _mk(rows, cols, mn, g):
    """A logical [rows x cols] bf16 view that is K-major (mn=0) or MN-major (mn=1)."""
    if mn:
        return torch.randn((cols, rows), generator=g, device="cuda").to(torch.bfloat16).T
    return torch.randn((rows, cols), generator=g, device="cuda").to(torch.bfloat16)


def _pitch_ok(M, N, K, a_mn, b_mn):
    """TMA needs 16-byte row pitches: an MN-major operand's pitch is its M (N)
    extent, a K-major one's is K (bf16: multiples of 8 elements)."""
    return not ((a_mn and M % 8) or (b_mn and N % 8) or (not a_mn and K % 8)
                or (not b_mn and K % 8))


_SHAPES = [(128, 256, 64), (256, 512, 256), (300, 4779, 200), (1366, 1024, 1000), (1, 8, 8),
           (130, 136, 72)]
_LAYOUTS = [(0, 0), (1, 0), (0, 1), (1, 1)]
_CASES = [s + l for s in _SHAPES for l in _LAYOUTS if _pitch_ok(*s, *l)]
_BAD = [s + l for s in _SHAPES for l in _LAYOUTS if not _pitch_ok(*s, *l)]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", _CASES)
def test_gemm_all_layouts(Lin, M, N, K, a_mn, b_mn):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + a_mn * 2 + b_mn)
    A = _mk(M, K, a_mn, g)
    B = _mk(N, K, b_mn, g)
    want = A.float() @ B.float().T
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    Lin.mm(A, B, out)
    torch.cuda.synchronize()
    assert rel(out, want) < 1e-5
    outb = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    Lin.mm(A, B, outb, alpha=0.5)
    assert rel(outb.float(), 0.5 * want) < 5e-3


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", _BAD[:4])
def test_gemm_rejects_unaligned_pitch(Lin, M, N, K, a_mn, b_mn):
    """Operands whose row pitch is not a multiple of 16 bytes are refused with a
    ValueError (TMA cannot map them), never computed wrongly."""
    g = torch.Generator(device="cuda").manual_seed(1)
    A, B = _mk(M, K, a_mn, g), _mk(N, K, b_mn, g)
    with pytest.raises(ValueError, match="16-byte"):
        Lin.mm(A, B, torch.empty((M, N), dtype=torch.float32, device="cuda"))


def test_gemm_epilogues_and_pitch(Lin):
    g = torch.Generator(device="cuda").manual_seed(5)
    M, N, K = 512, 4779, 256
    A = _mk(M, K, 0, g)
    B = _mk(N, K, 0, g)
    acc = A.float() @ B.float().T
    npad = (N + 7) // 8 * 8
    H = torch.empty((M, npad), dtype=torch.bfloat16, device="cuda")[:, :N]
    Y = torch.empty((M, npad), dtype=torch.bfloat16, device="cuda")[:, :N]
    Lin.mm(A, B, Y, epilogue="gelu", aux=H)
    assert rel(H.float(), acc) < 5e-3
    want = O.gelu(H.double().cpu().numpy())
    assert rel(Y.float().cpu(), torch.from_numpy(want)) < 5e-3
    D = torch.empty((M, npad), dtype=torch.bfloat16, device="cuda")[:, :N]
    Lin.mm(A, B, D, epilogue="dgelu", aux=H)
    want = acc.double().cpu().numpy() * O.gelu_grad(H.double().cpu().numpy())
    assert rel(D.float().cpu(), torch.from_numpy(want)) < 5e-3
    # output row pitch 2*N into an interleaved arena (the unit-major gradient layout)
    arena = torch.zeros((M, 2, N), dtype=torch.float32, device="cuda")
    Lin.mm(A, B, arena[:, 1, :])
    assert rel(arena[:, 1, :], acc) < 1e-5 and arena[:, 0, :].abs().max().item() == 0.0


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", [(3584, 4096, 8192, 1, 1),   # wgrad shape: 112 tiles
                                             (1366, 1024, 4000, 0, 0),   # ragged M and K
                                             (512, 2560, 2048, 1, 0)])
def test_gemm_split_k_tail(Lin, M, N, K, a_mn, b_mn):
    """The split-K tail (ntp_gemm_set_split_k) reproduces the whole-tile result
    for every epilogue: partials are summed in piece order, so repeated runs are
    bitwise identical, and the two schedules agree to fp32 rounding."""
    from paper_2504_06095_b200 import _lib
    L = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = _mk(M, K, a_mn, g)
    B = _mk(N, K, b_mn, g)
    acc = A.float() @ B.float().T
    res = {}
    try:
        for on in (1, 0):
            L.ntp_gemm_set_split_k(on)
            out = torch.empty((M, N), dtype=torch.float32, device="cuda")
            Lin.mm(A, B, out)
            again = torch.empty_like(out)
            Lin.mm(A, B, again)
            torch.cuda.synchronize()
            assert torch.equal(out, again)
            assert rel(out, acc) < 1e-5
            H = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
            Y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
            Lin.mm(A, B, Y, epilogue="gelu", aux=H)
            D = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
            Lin.mm(A, B, D, epilogue="dgelu", aux=H)
            want_d = acc.double().cpu().numpy() * O.gelu_grad(H.double().cpu().numpy())
            assert rel(D.float().cpu(), torch.from_numpy(want_d)) < 5e-3
            # fused red epilogue: the local copy and a "partner" copy both get alpha*acc
            loc = torch.zeros((M, N), dtype=torch.float32, device="cuda")
            far = torch.zeros((M, N), dtype=torch.float32, device="cuda")
            rb = torch.zeros(M, dtype=torch.int32, device="cuda")
            rr = torch.arange(M, dtype=torch.int32, device="cuda")
            Lin.mm_red(A, B, loc, 0.5, rb, rr, [far.data_ptr()], N)
            torch.cuda.synchronize()
            assert rel(loc, 0.5 * acc) < 1e-5 and rel(far, 0.5 * acc) < 1e-5
            res[on] = (out, H, Y, D)
    finally:
        L.ntp_gemm_set_split_k(1)
    assert rel(res[1][0], res[0][0]) < 2e-5  # different fp32 summation order
    # the last-arrival fixup path (no piece waits for the others) gives the same bits
    import ctypes
    fn = L.ntp_gemm_debug_split_window
    fn.argtypes = [ctypes.c_ulonglong]
    try:
        fn(0)
        out0 = torch.empty((M, N), dtype=torch.float32, device="cuda")
        Lin.mm(A, B, out0)
        torch.cuda.synchronize()
    finally:
        fn(250000)
    assert torch.equal(out0, res[1][0])
    for a, b in zip(res[1][1:], res[0][1:]):
        assert rel(a.float(), b.float()) < 1e-2
    assert rel(res[1][1].float(), acc) < 5e-3


def test_tp_mlp_forward_backward_vs_oracle(Lin):
    """TP4 comp layout of (1000, 4, 3): ragged, non-contiguous shards."""
    from paper_2504_06095_b200 import tpnumerics as T
    from paper_2504_06095_b200.shardmap import build_shard_map
    h, k, tok = 256, 1000, 512
    A, B = O.random_layer(h, k, seed=1)
    A, B = A / np.sqrt(h), B / np.sqrt(k)
    smap = build_shard_map(k, 4, 3)
    rng = np.random.default_rng(2)
    X = rng.standard_normal((tok, h))
    G = rng.standard_normal((tok, h))
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    r64 = lambda x: bf(x).double().numpy()  # noqa: E731
    A, B, X, G = r64(A), r64(B), r64(X), r64(G)
    for cols in (T.assignment_from_comp(smap), T.assignment_from_sync(smap)):
        shards = [Lin.MlpShard(A, B, c) for c in cols]
        Xd, Gd = bf(X).cuda(), bf(G).cuda()
        Z = Lin.mlp_forward_tp(Xd, shards)
        Zref = O.mlp_forward_dense(X, A, B)
        assert rel(Z.cpu(), torch.from_numpy(Zref)) < 2e-2
        rep = T.MlpReplica(T.MlpLayer(A, B), cols, dtype=torch.float32)
        Lin.mlp_backward_tp(Xd, shards, Gd, rep)
        want = O.mlp_backward_tp(X, A, B, G, cols)
        for u, (ga, gb) in zip(rep.units(), want):
            got_a, got_b = O.from_units(u, h)
            assert rel(torch.from_numpy(got_a), torch.from_numpy(ga)) < 2e-2
            assert rel(torch.from_numpy(got_b), torch.from_numpy(gb)) < 2e-2


def test_tensor_core_grads_then_sync(Lin):
    """Producer -> sync chain: tcgen05 wgrad writes the unit-major arenas that
    nonuniform_grad_sync reduces; the result matches the dense fp64 sum."""
    from paper_2504_06095_b200 import tpnumerics as T
    from paper_2504_06095_b200.shardmap import build_shard_map
    h, k, tok = 128, 600, 256
    A, B = O.random_layer(h, k, seed=3)
    A, B = A / np.sqrt(h), B / np.sqrt(k)
    smap = build_shard_map(k, 4, 3)
    rng = np.random.default_rng(4)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)  # noqa: E731
    r64 = lambda x: bf(x).double().numpy()  # noqa: E731
    A, B = r64(A), r64(B)
    X1, G1, X2, G2 = (r64(rng.standard_normal((tok, h))) for _ in range(4))
    layer = T.MlpLayer(A, B)
    reps = []
    for cols, X, G in ((T.assignment_from_comp(smap), X1, G1), (T.assignment_from_sync(smap), X2, G2)):
        shards = [Lin.MlpShard(A, B, c) for c in cols]
        rep = T.MlpReplica(layer, cols, dtype=torch.bfloat16)
        Lin.mlp_forward_tp(bf(X).cuda(), shards)
        Lin.mlp_backward_tp(bf(X).cuda(), shards, bf(G).cuda(), rep)
        reps.append(rep)
    T.nonuniform_grad_sync(reps[0], reps[1], smap)
    da1, db1 = O.mlp_backward(X1, A, B, G1)
    da2, db2 = O.mlp_backward(X2, A, B, G2)
    for rep in reps:
        da, db = rep.dense_grads()
        assert O.rel_err(da, da1 + da2) < 2e-2
        assert O.rel_err(db, db1 + db2) < 2e-2


def test_pdl_chains_match_stream_order(Lin):
    """Programmatic dependent launch (ntp_gemm_bf16_ex / MlpShard.backward(pdl=))
    changes only when GEMMs start: a multi-layer backward chained with
    "after"/"independent" launches gives the same bits as plain stream order,
    and so does the global ntp_gemm_set_pdl switch."""
    from paper_2504_06095_b200 import _lib
    h, k, tok, layers = 256, 1366, 512, 4
    rng = np.random.default_rng(7)
    shards, inputs = [], []
    for li in range(layers):
        A, B = O.random_layer(h, k, seed=10 + li)
        sh = Lin.MlpShard(A / np.sqrt(h), B / np.sqrt(k), np.arange(k))
        X = torch.from_numpy(rng.standard_normal((tok, h))).to(torch.bfloat16).cuda()
        G = torch.from_numpy(rng.standard_normal((tok, h))).to(torch.bfloat16).cuda()
        sh.forward(X, torch.empty((tok, h), dtype=torch.float32, device="cuda"))
        shards.append(sh)
        inputs.append((X, G))

    def run(pdl, global_pdl=0):
        _lib.load().ntp_gemm_set_pdl(global_pdl)
        try:
            out = [torch.zeros((k, 2, h), dtype=torch.float32, device="cuda") for _ in range(layers)]
            for li in reversed(range(layers)):
                mode = None if pdl is None else ("independent" if li < layers - 1 else "after")
                shards[li].backward(*inputs[li], out[li], pdl=mode)
            torch.cuda.synchronize()
            return out
        finally:
            _lib.load().ntp_gemm_set_pdl(0)

    want = run(None)
    for got in (run("chain"), run(None, global_pdl=1)):
        for a, b in zip(got, want):
            assert torch.equal(a, b)
    with pytest.raises(ValueError, match="unknown pdl mode"):
        Lin.mm(inputs[0][0], inputs[0][1], torch.empty((tok, tok), device="cuda"), pdl="soon")
