"""perfmodel.comm_comp_ratio (the reference's byte accounting, perfmodel.py:
244-278) on the C++ planner against values the reference itself computed
(tests/golden/comm_comp_ratio.json, made by tests/golden/make_golden.py)."""

import json
import os

import pytest

from paper_2504_06095_b200.perfmodel import ModelShape, comm_comp_ratio, reshard_bytes_per_layer

from conftest import GOLDEN


def _cases():
    with open(os.path.join(GOLDEN, "comm_comp_ratio.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['shape'][0]}-{c['n1']}-{c['n2']}")
def test_comm_comp_ratio_matches_reference(case):
    hidden, layers, heads, ffn = case["shape"]
    got = comm_comp_ratio(ModelShape(hidden=hidden, layers=layers, heads=heads, ffn=ffn),
                          case["n1"], case["n2"], case["pp"], case["local_batch"],
                          case["seq_len"], case["bytes_per_element"])
    assert got == case["ratio"]


def test_reshard_bytes_c2():
    """C2 (GPT-1.3B-shaped, TP4 -> TP3, bf16): the busiest rank of the pre-sync
    reshard is the offload rank, which sends all its 2048 MLP columns and 4
    heads per layer."""
    shape = ModelShape(hidden=2048, layers=24, heads=16, ffn=8192)
    assert reshard_bytes_per_layer(shape, 4, 3) == (2048 * 2 * 2048 + 4 * 4 * 2048 * 128) * 2
    assert reshard_bytes_per_layer(shape, 4, 4) == 0
