"""The reference's reshard byte accounting (perfmodel.py:223-278), on the C++
planner.

Only the volume accounting is on this path: it sizes
the gradient sync's bytes (a unit = an A column + a B row, 2*hidden elements;
a head = its four projection blocks, 4*hidden*head_dim).  The reference's
power and iteration-time models around it are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

from .shardmap import PRE_SYNC, build_reshard_plan, build_shard_map


@dataclass(frozen=True)
class ModelShape:
    """Transformer dimensions needed for volume accounting (perfmodel.py:223-241)."""

    hidden: int
    layers: int
    heads: int
    ffn: int | None = None

    @property
    def ffn_dim(self) -> int:
        return self.ffn if self.ffn is not None else 4 * self.hidden

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def params_per_layer(self) -> int:
        return 2 * self.hidden * self.ffn_dim + 4 * self.hidden * self.hidden


def reshard_bytes_per_layer(shape: ModelShape, n1: int, n2: int,
                            bytes_per_element: int = 2) -> int:
    """Busiest rank's one-direction reshard bytes for one layer: the larger of
    max columns sent / received of the pre-sync plan, for the MLP partition
    (k = ffn) and the head partition (k = heads)."""
    if n1 == n2:
        return 0

    def busiest(k: int) -> int:
        plan = build_reshard_plan(build_shard_map(k, n1, n2), PRE_SYNC)
        return max(plan.max_cols_sent, plan.max_cols_received)
    return (busiest(shape.ffn_dim) * 2 * shape.hidden
            + busiest(shape.heads) * 4 * shape.hidden * shape.head_dim) * bytes_per_element


def comm_comp_ratio(shape: ModelShape, n1: int, n2: int, pp: int, local_batch: int,
                    seq_len: int, bytes_per_element: int = 2) -> float:
    """Reshard bytes per GPU over backward FLOPs per GPU for one pipeline stage
    (perfmodel.py:244-278): the busiest rank's one-direction bytes summed over
    the stage's layers, over 4 x params per GPU x tokens."""
    if n1 == n2:
        return 0.0
    layers_per_stage = shape.layers / pp
    numerator = reshard_bytes_per_layer(shape, n1, n2, bytes_per_element) * layers_per_stage
    params_per_gpu = shape.params_per_layer() * layers_per_stage / n1
    return numerator / (4.0 * params_per_gpu * local_batch * seq_len)
