"""Synthetic gradient-sync workloads of BASELINE.json's configs, laid out in HBM.

A workload is a model's parameter-gradient set split into *segments*: per
layer, one MLP partition (k = ffn columns, unit = 2*hidden elements: A column
+ B row, perfmodel.py:269) and one attention partition (k = heads, unit =
4*hidden*head_dim elements: a head's q/k/v/o blocks, perfmodel.py:270-272).
Every segment is sharded by the reference's shard map (shardmap.py:141-182):
the healthy TP-n1 replica in comp layout, the degraded TP-n2 replica in sync
layout.  Each logical rank owns one flat arena holding its units of every
segment back to back, unit-major, so every unit is one contiguous run.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .plans import Plan, dtype_code
from .shardmap import build_shard_map
from .tpnumerics import build_pair_plan


@dataclass(frozen=True)
class ModelShape:
    """Volume accounting of perfmodel.py:223-241 (+ the layer count)."""

    name: str
    hidden: int
    ffn: int
    heads: int
    layers: int

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def segments(self):
        """[(kind, k, unit_elems)] for one layer."""
        segs = [("mlp", self.ffn, 2 * self.hidden)]
        if self.heads:
            segs.append(("attn", self.heads, 4 * self.hidden * self.head_dim))
        return segs

    def elems_per_layer(self) -> int:
        return sum(k * u for _, k, u in self.segments())

    def elems(self) -> int:
        return self.layers * self.elems_per_layer()


# BASELINE.json configs (SURVEY 8(d) choices: C2 16 heads, C4 32 heads / MHA)
C1 = ModelShape("mlp-h1024-ffn4096", 1024, 4096, 0, 1)
GPT_1_3B = ModelShape("gpt-1.3b", 2048, 8192, 16, 24)
LLAMA3_8B = ModelShape("llama3-8b-shaped", 4096, 14336, 32, 32)
SHAPES = {s.name: s for s in (GPT_1_3B, LLAMA3_8B, C1)}


@dataclass
class PairLayout:
    """Per-rank element counts and per-segment column lists of a TP-n1/TP-n2 pair."""

    shape: ModelShape
    n1: int
    n2: int
    layers: int
    h_elems: list = field(default_factory=list)
    r_elems: list = field(default_factory=list)
    segs: list = field(default_factory=list)  # (k, unit, h_cols, r_cols, h_base, r_base)

    @property
    def elems(self) -> int:
        return sum(self.h_elems)


def pair_layout(shape: ModelShape, n1: int, n2: int, layers: int | None = None) -> PairLayout:
    layers = shape.layers if layers is None else layers
    lay = PairLayout(shape, n1, n2, layers)
    h_base = np.zeros(n1, dtype=np.int64)
    r_base = np.zeros(n2, dtype=np.int64)
    seg_kinds = shape.segments()
    maps = {k: build_shard_map(k, n1, n2) for _, k, _ in seg_kinds}
    for _ in range(layers):
        for _, k, unit in seg_kinds:
            smap = maps[k]
            hc = [smap.comp_columns(r) for r in range(n1)]
            rc = [smap.sync_columns(r) for r in range(n2)]
            lay.segs.append((k, unit, hc, rc, h_base.copy(), r_base.copy()))
            h_base += np.array([len(c) for c in hc]) * unit
            r_base += np.array([len(c) for c in rc]) * unit
    lay.h_elems = h_base.tolist()
    lay.r_elems = r_base.tolist()
    return lay


def build_plan(lay: PairLayout, dtype, h_bufs=None, r_bufs=None, seg_filter=None) -> Plan:
    """One plan over all segments; optional seg_filter(index) selects segments."""
    plan = Plan(dtype_code(dtype))
    for i, (k, unit, hc, rc, hb, rb) in enumerate(lay.segs):
        if seg_filter is not None and not seg_filter(i):
            continue
        build_pair_plan(hc, rc, k, unit, plan.dtype, h_base=hb, r_base=rb, h_bufs=h_bufs,
                        r_bufs=r_bufs, plan=plan)
    return plan.finalize()


def busiest_bytes(lay: PairLayout, elem_bytes: int) -> int:
    """B_busiest: the GPU that ends owning the most elements must
    receive and send that many elements once per direction."""
    return max(max(lay.h_elems), max(lay.r_elems)) * elem_bytes


def layer_pieces(lay: PairLayout, dtype, device: int, layers_per_piece: int = 1,
                 segs_per_piece: int | None = None):
    """Per-layer (or per-segment: segs_per_piece=1 splits a layer into its MLP
    and attention parts) plans + the arena element ranges each touches
    (HostSync pieces).  Segments are contiguous in every arena, so a piece is
    one element range per arena."""
    nseg = len(lay.shape.segments())
    step = segs_per_piece if segs_per_piece else nseg * layers_per_piece
    pieces = []
    n1 = lay.n1
    total = lay.layers * nseg
    for s0 in range(0, total, step):
        idx = range(s0, min(total, s0 + step))
        plan = build_plan(lay, dtype, seg_filter=lambda i, s=idx: i in s).upload(device)
        ranges = []
        for side, count in ((0, n1), (1, lay.n2)):
            for a in range(count):
                lo = int(lay.segs[idx[0]][4 + side][a])
                last = lay.segs[idx[-1]]
                hi = int(last[4 + side][a]) + len(last[2 + side][a]) * last[1]
                ranges.append((a + side * n1, lo, hi))
        pieces.append((plan, ranges))
    return pieces
