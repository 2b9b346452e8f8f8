"""The C planner (libntp_b200.so via paper_2504_06095_b200.shardmap) is
bit-exact with the reference's shard algebra (fixtures from the reference)
and with the oracle; the reference's own property tests run against it."""

import hashlib
import json
import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O
from paper_2504_06095_b200.shardmap import (
    POST_SYNC, PRE_SYNC, ShardMap, apply_plan, attention_head_partition, build_reshard_plan,
    build_shard_map, interval_overlaps, naive_contiguous_sync_volumes,
)

from conftest import GOLDEN


def _fx():
    with open(os.path.join(GOLDEN, "shardmaps.json")) as f:
        return json.load(f)


def _digest(smap, pre, post):
    doc = {"map": smap.to_json_dict(), "pre": pre.to_json_dict(), "post": post.to_json_dict()}
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()


def test_full_fixtures_bit_exact():
    for case in _fx()["full"]:
        smap = build_shard_map(case["k"], case["n1"], case["n2"])
        assert smap.to_json_dict() == case["map"]
        pre = build_reshard_plan(smap, PRE_SYNC)
        post = build_reshard_plan(smap, POST_SYNC)
        assert pre.to_json_dict() == case["pre"]
        assert post.to_json_dict() == case["post"]
        assert [pre.total_cols_moved, pre.max_cols_sent, pre.max_cols_received] == case["pre_stats"]
        assert [post.total_cols_moved, post.max_cols_sent, post.max_cols_received] == case["post_stats"]
        got = naive_contiguous_sync_volumes(case["k"], case["n1"], case["n2"])
        assert [[list(p) for p in r] for r in got] == case["naive"]


def test_crit02_digests_bit_exact():
    """The 1000 random triples of acceptance criterion 02 (rng seed 0)."""
    for k, n1, n2, dig in _fx()["crit02"]:
        smap = build_shard_map(k, n1, n2)
        pre = build_reshard_plan(smap, PRE_SYNC)
        post = build_reshard_plan(smap, POST_SYNC)
        assert _digest(smap, pre, post) == dig, (k, n1, n2)
        assert np.array_equal(apply_plan(smap.comp_rank, pre), smap.sync_rank)
        assert np.array_equal(apply_plan(smap.sync_rank, post), smap.comp_rank)


def test_big_configs_bit_exact():
    for case in _fx()["big"]:
        smap = build_shard_map(case["k"], case["n1"], case["n2"])
        pre = build_reshard_plan(smap, PRE_SYNC)
        post = build_reshard_plan(smap, POST_SYNC)
        assert _digest(smap, pre, post) == case["digest"]
        assert [pre.total_cols_moved, pre.max_cols_sent, pre.max_cols_received] == case["pre_stats"]


def test_head_partition_matches_reference():
    for case in _fx()["heads"]:
        counts, imb = attention_head_partition(case["heads"], case["n"])
        assert counts.tolist() == case["counts"]
        assert imb == case["imbalance"]
    with pytest.raises(ValueError, match="exceeds head count"):
        attention_head_partition(3, 4)
    with pytest.raises(ValueError, match="must be positive"):
        attention_head_partition(0, 1)


def test_invalid_triples_same_messages():
    for k, n1, n2, msg in _fx()["errors"]:
        with pytest.raises(ValueError) as ei:
            build_shard_map(k, n1, n2)
        assert str(ei.value) == msg
    with pytest.raises(ValueError, match="direction must be"):
        build_reshard_plan(build_shard_map(8, 4, 2), "sideways")


def test_apply_plan_rejects_non_owned_columns():
    smap = build_shard_map(12, 4, 3)
    pre = build_reshard_plan(smap, PRE_SYNC)
    with pytest.raises(ValueError, match="names columns not owned by"):
        apply_plan(smap.sync_rank, pre)  # pre must start from comp ownership


@st.composite
def triples(draw):
    n1 = draw(st.integers(1, 16))
    n2 = draw(st.integers(1, n1))
    k = draw(st.integers(n1, 512))
    return k, n1, n2


@given(triples())
@settings(max_examples=200, deadline=None)
def test_planner_equals_oracle(t):
    k, n1, n2 = t
    smap = build_shard_map(k, n1, n2)
    comp, sync = O.shard_map(k, n1, n2)
    assert np.array_equal(smap.comp_rank, comp)
    assert np.array_equal(smap.sync_rank, sync)
    for d in (PRE_SYNC, POST_SYNC):
        got = [(t.src, t.dst, t.cols) for t in build_reshard_plan(smap, d).transfers]
        assert got == O.reshard_plan(comp, sync, n1, d)
    assert naive_contiguous_sync_volumes(k, n1, n2) == O.naive_overlaps(k, n1, n2)


@given(triples())
@settings(max_examples=200, deadline=None)
def test_reference_properties(t):
    """test_shardmap.py:27-98 properties on the C planner."""
    k, n1, n2 = t
    smap = build_shard_map(k, n1, n2)
    comp = np.concatenate([smap.comp_columns(r) for r in range(n1)])
    assert np.array_equal(np.sort(comp), np.arange(k))
    assert smap.comp_counts().max() - smap.comp_counts().min() <= 1
    assert smap.sync_counts().max() - smap.sync_counts().min() <= 1
    start = 0
    for r in range(n2):
        cols = smap.sync_columns(r)
        assert np.array_equal(cols, np.arange(start, start + len(cols)))
        start += len(cols)
        own = set(smap.comp_columns(r))
        keep = [c for c in cols if c in own]
        assert keep == list(cols[: len(keep)])
    pre = build_reshard_plan(smap, PRE_SYNC)
    post = build_reshard_plan(smap, POST_SYNC)
    assert np.array_equal(apply_plan(smap.comp_rank, pre), smap.sync_rank)
    assert np.array_equal(apply_plan(smap.sync_rank, post), smap.comp_rank)
    links = post.link_volumes()
    for src in range(n2):
        vols = [links.get((src, dst), 0) for dst in range(n2, n1)]
        if vols:
            assert max(vols) - min(vols) <= 1


@given(st.integers(1, 3000), st.integers(1, 40), st.integers(1, 40))
@settings(max_examples=200, deadline=None)
def test_interval_overlaps_tile_the_range(k, a, b):
    if a > k or b > k:
        with pytest.raises(ValueError):
            interval_overlaps(k, a, b)
        return
    q = interval_overlaps(k, a, b)
    assert q[0][2] == 0 and sum(x[3] for x in q) == k
    for (s0, d0, p0, l0), (s1, d1, p1, l1) in zip(q, q[1:]):
        assert p0 + l0 == p1 and (s1, d1) > (s0, d0)
    src = np.concatenate([[s] * ln for s, _, _, ln in q])
    dst = np.concatenate([[d] * ln for _, d, _, ln in q])
    sizes = k // a + (np.arange(a) < k % a)
    assert np.array_equal(src, np.repeat(np.arange(a), sizes))
    sizes = k // b + (np.arange(b) < k % b)
    assert np.array_equal(dst, np.repeat(np.arange(b), sizes))
    if b <= a:  # the naive planner is the n2 <= n1 special case
        naive = naive_contiguous_sync_volumes(k, a, b)
        flat = [(d, s, ln) for s, d, _, ln in q]
        assert flat == [(i, h, ov) for i, r in enumerate(naive) for h, ov in r]


def test_contrast_case():
    smap = build_shard_map(12000, 32, 30)
    assert set(smap.comp_counts()) == {375} and set(smap.sync_counts()) == {400}
    post = build_reshard_plan(smap, POST_SYNC)
    assert (post.total_cols_moved, post.max_cols_sent, post.max_cols_received) == (750, 25, 375)


def test_json_round_trip():
    smap = build_shard_map(100, 7, 5)
    again = ShardMap.from_json_dict(json.loads(smap.to_json()))
    assert np.array_equal(again.comp_rank, smap.comp_rank)
    plan = build_reshard_plan(smap, PRE_SYNC)
    assert json.loads(plan.to_json())["direction"] == PRE_SYNC
