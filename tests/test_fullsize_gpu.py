"""Full-size parity: the exact plans bench.py times, every segment vs the oracle.

The bench's N=1 step is ONE launch of the default (AUTO -> TMA-bulk) sync
kernel over a whole model's gradient: GPT-1.3B-shaped (24 layers x (MLP +
attention) segments, 7 arenas, 147 480 chunks) in bf16.  Here that same plan
(``workloads.build_plan(pair_layout(...))``) runs once on fresh N(0,1) arenas
and every segment of every layer is compared with the fp64 oracle
(oracle.nonuniform_sync, tpnumerics.py:289-356) on the same bf16-rounded
inputs, with the arena layout taken from the oracle's own shard map.  Tolerances
(north_star): bf16 <= 2e-2, fp32 <= 1e-6 Frobenius relative error per segment;
the healthy and reduced copies of every unit must also be bit-identical.
"""

import pytest
import torch

import bench

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import workloads
    return workloads


def _run(W, shape, layers, dtype, kernel=0, weights=(bench.W_H, bench.W_R)):
    from paper_2504_06095_b200 import _lib
    L = _lib.load()
    lay = W.pair_layout(shape, 4, 3, layers=layers)
    plan = W.build_plan(lay, dtype).upload(0)
    arenas = [torch.empty(e, dtype=dtype, device="cuda") for e in lay.h_elems + lay.r_elems]
    _lib.check(L.ntp_set_option(0, kernel))  # NTP_OPT_SYNC_KERNEL (0 = AUTO, as the bench)
    try:
        res = bench.check_pair_arenas(shape.hidden, shape.ffn, shape.heads, layers, plan, arenas,
                                      dtype, lay.h_elems, lay.r_elems, weights=weights)
    finally:
        L.ntp_set_option(0, 0)
    del arenas
    torch.cuda.empty_cache()
    return res


def test_c2_full_step_every_segment(W):
    """BASELINE configs[1] exactly as benchmarked: 24 layers, bf16, AUTO kernel."""
    res = _run(W, W.GPT_1_3B, W.GPT_1_3B.layers, torch.bfloat16)
    assert res["ok"] and res["segments"] == 48 and res["chunks"] == 147480, res


def test_c4_four_layers_every_segment(W):
    """BASELINE configs[3] shape (Llama-3-8B, h4096, ffn14336, 32 heads), 4 layers."""
    res = _run(W, W.LLAMA3_8B, 4, torch.bfloat16)
    assert res["ok"] and res["segments"] == 8, res


@pytest.mark.parametrize("kernel", [1, 2, 3], ids=["ldg", "bulk4", "bulk3x2"])
def test_c2_two_layers_each_kernel_variant(W, kernel):
    res = _run(W, W.GPT_1_3B, 2, torch.bfloat16, kernel=kernel)
    assert res["ok"], res


def test_c1_fp32(W):
    """BASELINE configs[0] (the CPU reference's own shape) in fp32, <= 1e-6."""
    res = _run(W, W.C1, 1, torch.float32)
    assert res["ok"] and res["max_rel_err"] <= 1e-6, res


def test_c1_fp16(W):
    """fp16 arenas (the library accepts NTP_F16): fp32 accumulate, <= 2e-3."""
    res = _run(W, W.C1, 1, torch.float16)
    assert res["ok"], res


@pytest.mark.parametrize("weights", [(1.0, 1.0), (0.5, 0.5)], ids=["sum", "mean"])
def test_c2_layer_sum_and_mean_weights(W, weights):
    res = _run(W, W.GPT_1_3B, 1, torch.bfloat16, weights=weights)
    assert res["ok"], res
