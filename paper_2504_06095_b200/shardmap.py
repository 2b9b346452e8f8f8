"""Shard-map algebra with the reference's API, computed by the C planner.

Drop-in for ``ntpsim.shardmap`` (pkg/src/ntpsim/shardmap.py): same names,
argument meaning, return types, JSON shapes and ValueError texts.  The integer
work runs in libntp_b200.so (``ntp_shard_map`` & co., include/ntp_b200.h);
this module only wraps arrays and records.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _lib

PRE_SYNC = "pre_sync"    # shardmap.py:19
POST_SYNC = "post_sync"  # shardmap.py:20
_DIRECTIONS = {PRE_SYNC: _lib.NTP_PRE_SYNC, POST_SYNC: _lib.NTP_POST_SYNC}


@dataclass(frozen=True)
class ShardMap:
    """Column -> (comp rank, sync rank) assignment of one NTP pair (shardmap.py:30-81).

    ``comp_rank[j]`` in [0, n1) computes with column j; ``sync_rank[j]`` in
    [0, n2) holds its gradient during the pairwise reduce.
    """

    k: int
    n1: int
    n2: int
    comp_rank: np.ndarray
    sync_rank: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "comp_rank", _lib.i64(self.comp_rank))
        object.__setattr__(self, "sync_rank", _lib.i64(self.sync_rank))

    def comp_columns(self, rank: int) -> np.ndarray:
        return np.flatnonzero(self.comp_rank == rank)

    def sync_columns(self, rank: int) -> np.ndarray:
        return np.flatnonzero(self.sync_rank == rank)

    def comp_counts(self) -> np.ndarray:
        return np.bincount(self.comp_rank, minlength=self.n1)

    def sync_counts(self) -> np.ndarray:
        return np.bincount(self.sync_rank, minlength=self.n2)

    def to_json_dict(self) -> dict:
        return {"k": self.k, "n1": self.n1, "n2": self.n2,
                "comp_rank": self.comp_rank.tolist(), "sync_rank": self.sync_rank.tolist()}

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())

    @classmethod
    def from_json_dict(cls, d: dict) -> "ShardMap":
        return cls(k=int(d["k"]), n1=int(d["n1"]), n2=int(d["n2"]),
                   comp_rank=_lib.i64(d["comp_rank"]), sync_rank=_lib.i64(d["sync_rank"]))


@dataclass(frozen=True)
class Transfer:
    """Columns moved over one ordered link (shardmap.py:84-88)."""

    src: int
    dst: int
    cols: tuple[int, ...]


@dataclass(frozen=True)
class ReshardPlan:
    """Per-link column moves between comp and sync layouts (shardmap.py:91-129)."""

    direction: str
    transfers: tuple[Transfer, ...]

    @property
    def total_cols_moved(self) -> int:
        return sum(len(t.cols) for t in self.transfers)

    def _per(self, attr: str) -> dict[int, int]:
        acc: dict[int, int] = {}
        for t in self.transfers:
            r = getattr(t, attr)
            acc[r] = acc.get(r, 0) + len(t.cols)
        return acc

    @property
    def max_cols_sent(self) -> int:
        return max(self._per("src").values(), default=0)

    @property
    def max_cols_received(self) -> int:
        return max(self._per("dst").values(), default=0)

    def link_volumes(self) -> dict[tuple[int, int], int]:
        return {(t.src, t.dst): len(t.cols) for t in self.transfers}

    def to_json_dict(self) -> dict:
        return {"direction": self.direction,
                "transfers": [{"src": t.src, "dst": t.dst, "cols": list(t.cols)}
                              for t in self.transfers]}

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())

    @cached_property
    def triples(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Flattened (src, dst, col) arrays in transfer order (the C ABI form)."""
        if not self.transfers:
            e = np.empty(0, dtype=np.int64)
            return e, e.copy(), e.copy()
        src = np.concatenate([np.full(len(t.cols), t.src, dtype=np.int64) for t in self.transfers])
        dst = np.concatenate([np.full(len(t.cols), t.dst, dtype=np.int64) for t in self.transfers])
        col = np.concatenate([_lib.i64(t.cols) for t in self.transfers])
        return src, dst, col


def build_shard_map(k: int, n1: int, n2: int) -> ShardMap:
    """Algorithm 1 (prose reading), shardmap.py:141-182, via ``ntp_shard_map``."""
    L = _lib.load()
    n = max(int(k), 0)
    comp = np.empty(n, dtype=np.int64)
    sync = np.empty(n, dtype=np.int64)
    _lib.check(L.ntp_shard_map(int(k), int(n1), int(n2), _lib.p64(comp), _lib.p64(sync)))
    return ShardMap(k=int(k), n1=int(n1), n2=int(n2), comp_rank=comp, sync_rank=sync)


def build_reshard_plan(smap: ShardMap, direction: str) -> ReshardPlan:
    """Comp->sync (pre) or sync->comp (post) transfers, shardmap.py:185-206."""
    if direction not in _DIRECTIONS:
        raise ValueError(f"direction must be {PRE_SYNC!r} or {POST_SYNC!r}, got {direction!r}")
    L = _lib.load()
    k = smap.k
    src, dst, col = (np.empty(k, dtype=np.int64) for _ in range(3))
    n = _lib.check(L.ntp_reshard_plan(_lib.p64(smap.comp_rank), _lib.p64(smap.sync_rank), k,
                                      max(smap.n1, 1), _DIRECTIONS[direction], _lib.p64(src),
                                      _lib.p64(dst), _lib.p64(col)))
    transfers = []
    if n:
        src, dst, col = src[:n], dst[:n], col[:n]
        key = src * max(smap.n1, 1) + dst
        cuts = np.flatnonzero(np.diff(key)) + 1
        for lo, hi in zip(np.r_[0, cuts], np.r_[cuts, n]):
            transfers.append(Transfer(src=int(src[lo]), dst=int(dst[lo]),
                                      cols=tuple(col[lo:hi].tolist())))
    return ReshardPlan(direction=direction, transfers=tuple(transfers))


def apply_plan(ownership: np.ndarray, plan: ReshardPlan) -> np.ndarray:
    """Replay a plan on a column->rank vector (shardmap.py:209-217)."""
    out = np.array(ownership, dtype=np.int64, copy=True)
    src, dst, col = plan.triples
    _lib.check(_lib.load().ntp_apply_plan(_lib.p64(out), len(out), _lib.p64(src), _lib.p64(dst),
                                          _lib.p64(col), len(col)))
    return out


def naive_contiguous_sync_volumes(k: int, n1: int, n2: int) -> list[list[tuple[int, int]]]:
    """Contiguous-vs-contiguous overlap sizes (shardmap.py:220-245)."""
    L = _lib.load()
    pairs = np.empty(2 * (max(n1, 0) + max(n2, 0)) + 2, dtype=np.int64)
    per = np.empty(max(n2, 1), dtype=np.int64)
    _lib.check(L.ntp_naive_overlaps(int(k), int(n1), int(n2), _lib.p64(pairs), _lib.p64(per)))
    out, at = [], 0
    for i in range(n2):
        c = int(per[i])
        out.append([(int(pairs[2 * q]), int(pairs[2 * q + 1])) for q in range(at, at + c)])
        at += c
    return out


def interval_overlaps(k: int, n_src: int, n_dst: int) -> list[tuple[int, int, int, int]]:
    """(src_rank, dst_rank, start, length) pieces between contiguous TP-n_src and
    TP-n_dst partitions of k: the TP-k -> TP-(k-f) planner (no reference
    function; generalises naive_contiguous_sync_volumes, shardmap.py:220-245)."""
    quads = np.empty(4 * (n_src + n_dst) + 4, dtype=np.int64)
    n = _lib.check(_lib.load().ntp_interval_overlaps(int(k), int(n_src), int(n_dst),
                                                     _lib.p64(quads)))
    return [tuple(int(v) for v in quads[4 * i:4 * i + 4]) for i in range(n)]


def attention_head_partition(heads: int, n: int) -> tuple[np.ndarray, float]:
    """Balanced contiguous head counts and imbalance factor (shardmap.py:248-260)."""
    counts = np.empty(max(int(n), 1), dtype=np.int64)
    imb = ctypes.c_double(0.0)
    _lib.check(_lib.load().ntp_head_partition(int(heads), int(n), _lib.p64(counts),
                                              ctypes.byref(imb)))
    return counts[: int(n)], float(imb.value)
