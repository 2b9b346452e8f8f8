"""Device canaries: the kernels write only the bytes their plans and views own.

compute-sanitizer is closed on the B200 pool (it left GPUs needing a reset),
so out-of-bounds writes are caught here directly: every buffer a kernel
touches sits between guard regions filled with a byte pattern, and views with
a row pitch wider than their rows keep the pattern in the gaps.  After the
launch every guard byte must be intact.  tests/test_plan_check.py checks the
plans statically (bounds, no element written twice).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 1 << 16  # bytes each side
PATTERN = 0xA5


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import _lib
    return _lib.load()


def guarded(numel, dtype):
    """(tensor of numel elements inside a guarded byte buffer, raw buffer)."""
    eb = torch.empty(0, dtype=dtype).element_size()
    raw = torch.full((2 * GUARD + numel * eb,), PATTERN, dtype=torch.uint8, device="cuda")
    t = raw[GUARD:GUARD + numel * eb].view(dtype)
    return t, raw


def guards_intact(raw, numel_bytes):
    return bool(torch.all(raw[:GUARD] == PATTERN)) and bool(torch.all(raw[GUARD + numel_bytes:] == PATTERN))


@pytest.mark.parametrize("variant", [0, 1, 2, 3], ids=["auto", "ldg", "bulk4", "bulk3x2"])
@pytest.mark.parametrize("case", ["c2_two_layers_bf16", "odd_fp32_scalar"])
def test_sync_kernels_stay_inside_arenas(lib, variant, case):
    from paper_2504_06095_b200.plans import OPS, tensor_ptrs
    from paper_2504_06095_b200.workloads import GPT_1_3B, ModelShape, build_plan, pair_layout
    if case == "c2_two_layers_bf16":
        lay, dt = pair_layout(GPT_1_3B, 4, 3, layers=2), torch.bfloat16
    else:  # 2*hidden = 66 elements: units not 16-byte aligned -> scalar plan
        lay, dt = pair_layout(ModelShape("odd", 33, 601, 0, 2), 4, 3), torch.float32
    plan = build_plan(lay, dt).upload(0)
    elems = list(lay.h_elems) + list(lay.r_elems)
    bufs = [guarded(e, dt) for e in elems]
    for t, _ in bufs:
        t.copy_(torch.randn(t.numel(), device="cuda").to(dt))
    lib.ntp_set_option(0, variant)
    try:
        plan.grad_sync(tensor_ptrs([t for t, _ in bufs]), OPS["weighted"], 4 / 7, 3 / 7)
        torch.cuda.synchronize()
    finally:
        lib.ntp_set_option(0, 0)
    eb = torch.empty(0, dtype=dt).element_size()
    assert all(guards_intact(raw, e * eb) for (_, raw), e in zip(bufs, elems))


def test_uniform_and_reduce_into_stay_inside(lib):
    import ctypes

    from paper_2504_06095_b200 import _lib
    n = 1000003  # odd: vector body + scalar tail
    bufs = [guarded(n, torch.float32) for _ in range(3)]
    for t, _ in bufs:
        t.normal_()
    w = (ctypes.c_double * 3)(0.5, 0.25, 0.25)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.ntp_uniform_sync(_lib.ptr_array([t.data_ptr() for t, _ in bufs]), 3, n,
                                    _lib.NTP_F32, 2, w, s))
    dst = [guarded(n, torch.float32) for _ in range(2)]
    _lib.check(lib.ntp_reduce_into(_lib.ptr_array([t.data_ptr() for t, _ in bufs]), 3, n,
                                   _lib.NTP_F32, _lib.ptr_array([t.data_ptr() for t, _ in dst]), 2,
                                   s))
    torch.cuda.synchronize()
    assert all(guards_intact(raw, n * 4) for _, raw in bufs + dst)
    want = bufs[0][0] + bufs[1][0] + bufs[2][0]
    assert all(torch.equal(t, want) for t, _ in dst)


@pytest.mark.parametrize("n", [4779, 3584, 600])
def test_gemms_write_only_their_views(lib, n):
    """The five per-rank GEMMs of a TP shard write only their output views:
    H/Y leave the padding columns of their pitch alone; the dB GEMM leaves the
    A half of every unit untouched and the dA GEMM the B half; every buffer's
    guards stay intact."""
    from paper_2504_06095_b200.linear import MlpShard, _pad8, mm
    h, T = 512, 384
    rng = np.random.default_rng(n)
    A = rng.standard_normal((h, n)) / np.sqrt(h)
    B = rng.standard_normal((n, h)) / np.sqrt(n)
    sh = MlpShard(A, B, np.arange(n))
    X = torch.randn((T, h), device="cuda").to(torch.bfloat16)
    G = torch.randn((T, h), device="cuda").to(torch.bfloat16)
    npad = _pad8(n) + 8  # a pitch wider than the rows
    Hb, Hraw = guarded(T * npad, torch.bfloat16)
    Yb, Yraw = guarded(T * npad, torch.bfloat16)
    H, Y = Hb.view(T, npad)[:, :n], Yb.view(T, npad)[:, :n]
    mm(X, sh.W[:, 0, :], Y, epilogue="gelu", aux=H)
    Zb, Zraw = guarded(T * h, torch.float32)
    mm(Y, sh.W[:, 1, :].T, Zb.view(T, h))
    Db, Draw = guarded(T * npad, torch.bfloat16)
    D = Db.view(T, npad)[:, :n]
    mm(G, sh.W[:, 1, :], D, epilogue="dgelu", aux=H)
    gb, graw = guarded(n * 2 * h, torch.float32)
    grads = gb.view(n, 2, h)
    mm(Y.T, G.T, grads[:, 1, :])
    torch.cuda.synchronize()
    untouched_a = graw[GUARD:GUARD + n * 2 * h * 4].view(n, 2, h * 4)[:, 0, :]
    assert bool(torch.all(untouched_a == PATTERN)), "dB GEMM wrote into the A half"
    dB = grads[:, 1, :].clone()
    mm(D.T, X.T, grads[:, 0, :])
    torch.cuda.synchronize()
    assert torch.equal(grads[:, 1, :], dB), "dA GEMM wrote into the B half"
    for raw, nbytes in ((Hraw, T * npad * 2), (Yraw, T * npad * 2), (Zraw, T * h * 4),
                        (Draw, T * npad * 2), (graw, n * 2 * h * 4)):
        assert guards_intact(raw, nbytes)
    for buf in (Hraw, Yraw, Draw):
        pad = buf[GUARD:GUARD + T * npad * 2].view(T, npad * 2)[:, n * 2:]
        assert bool(torch.all(pad == PATTERN)), "a GEMM wrote into its output's pitch padding"


@pytest.mark.parametrize("h", [40, 72, 512])
def test_wgrad_into_bf16_arena_keeps_neighbouring_half_units(lib, h):
    """Unit-major bf16 arena [n, 2, h]: the dB GEMM writes rows of h elements
    with a 2h pitch, next to the same unit's (and the next unit's) A half,
    which must stay untouched.  (Here a row always ends on a 16-byte boundary,
    because the G operand's own pitch, h elements, must be 16-byte aligned for
    TMA; the H/Y/D case above is the one whose rows end mid-granule.)"""
    from paper_2504_06095_b200.linear import mm
    n, T = 104, 256  # Y's pitch (n elements) must be 16-byte aligned for TMA
    X = torch.randn((T, h), device="cuda").to(torch.bfloat16)
    Y = torch.randn((T, n), device="cuda").to(torch.bfloat16)
    G = torch.randn((T, h), device="cuda").to(torch.bfloat16)
    gb, graw = guarded(n * 2 * h, torch.bfloat16)
    grads = gb.view(n, 2, h)
    mm(Y.T, G.T, grads[:, 1, :])
    torch.cuda.synchronize()
    a_half = graw[GUARD:GUARD + n * 2 * h * 2].view(n, 2, h * 2)[:, 0, :]
    assert bool(torch.all(a_half == PATTERN)), "dB GEMM spilled into the A half"
    want = (Y.float().T @ G.float())
    assert torch.allclose(grads[:, 1, :].float(), want, rtol=2e-2, atol=2e-2 * want.abs().max().item())
    assert guards_intact(graw, n * 2 * h * 2)
    del X
