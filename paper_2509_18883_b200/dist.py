"""Data parallelism over the hot path.

Fusion shards by parameter range: the global item list (every tensor cut into RLK_FUSION_ITEM-element
items from its own start) is split into world-size contiguous ranges balanced by element count
(`FusionLayout.partition`).  Each rank holds only its range of base + experts and writes only its
range of the output.  The one exchange is the all_reduce of the f64 norm partials between K1 and
finalize, restricted to the item rows of the tensors that are split over ranks (a tensor held whole by
one rank needs no exchange) -- every (item, expert) slot is produced by exactly one rank and is
exactly zero elsewhere, so the NCCL sum is exact and the norms (hence scales, masks, erase decisions
and outputs) are bit-identical at every world size.  With `FusionLayout.partition_striped` (the default here) the
embedding-sized tensors are cut into one stripe per rank, so each rank draws only the dropout keep
bits of its own index ranges and no bitmap crosses GPUs.  FusionStats counters are summed by a second (int64) all_reduce
only when statistics are requested.

The GRPO loss shards by response; per-group token-term sums are all-reduced (objective.grpo_forward).

The collectives here take torch tensors and a process group, so the same code runs over NCCL on
GPUs and over gloo on CPU tensors (tests/test_dist_cpu.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import torch

from .fusion import FusionCall, FusionConfig, FusionLayout, FusionStats, Piece


def allreduce_partials(partials: torch.Tensor, group) -> torch.Tensor:
    """Exact sum of disjointly-written f64 partial slots (x + 0 == x, whatever the reduction order)."""
    import torch.distributed as dist
    if group is not None:
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    return partials


def allreduce_counts(counts: torch.Tensor, group) -> torch.Tensor:
    import torch.distributed as dist
    if group is not None:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def rank_pieces(layout: FusionLayout, world: int, rank: int) -> list[tuple[int, int, int]]:
    """This rank's (tensor, lo, hi) element ranges (big tensors striped over the ranks)."""
    return layout.partition_striped(world, rank)


def shard_state_dicts(base: Mapping[str, torch.Tensor], experts: Sequence[Mapping[str, torch.Tensor]], world: int,
                      rank: int, out_dtype: torch.dtype | None = None):
    """Slice full state dicts (any device) into this rank's pieces on the current CUDA device.

    Returns (names, layout, pieces).  A real deployment would read only its ranges from storage
    (loader.py); this helper is for checkpoints that every rank can see."""
    names = list(base.keys())
    layout = FusionLayout([base[k].numel() for k in names])
    dev = torch.device("cuda", torch.cuda.current_device())
    pieces = []
    for t, lo, hi in layout.partition_striped(world, rank):
        name = names[t]
        b = base[name].reshape(-1)[lo:hi].to(dev).contiguous()
        es = [e[name].reshape(-1)[lo:hi].to(dev).contiguous() for e in experts]
        out = torch.empty(hi - lo, dtype=out_dtype or b.dtype, device=dev)
        pieces.append(Piece(t, lo, b, es, out))
    return names, layout, pieces


@dataclass
class ShardedFusion:
    """A parameter-range-sharded fusion on one rank (one FusionCall, reusable across steps)."""

    names: list[str]
    layout: FusionLayout
    pieces: list[Piece]
    call: FusionCall
    weights: tuple[float, ...]
    group: object = None

    @staticmethod
    def build(names, layout, pieces, n_experts: int, cfg: FusionConfig, group=None, stream=None) -> "ShardedFusion":
        weights = cfg.merge_weights or tuple(1.0 / n_experts for _ in range(n_experts))
        call = FusionCall(pieces, layout, n_experts, cfg, group=group, stream=stream)
        return ShardedFusion(list(names), layout, list(pieces), call, tuple(weights), group)

    def run(self) -> "ShardedFusion":
        self.call.run(self.weights)
        return self

    def stats(self) -> dict[str, FusionStats]:
        """Global FusionStats per tensor: counters summed over ranks; each tensor's sum of squares and
        scale from its owner rank (the only one contributing a non-zero row: exact sums)."""
        c = self.call
        counters = allreduce_counts(c.counters.clone(), self.group)
        sumsq, scale = c.sumsq, c.scale
        if c._owner is not None:
            own = c._owner.view(-1, 1)
            sumsq = allreduce_partials(torch.where(own, c.sumsq, torch.zeros_like(c.sumsq)), self.group)
            scale = allreduce_partials(torch.where(own, c.scale, torch.zeros_like(c.scale)), self.group)
        saved = c.counters, c.sumsq, c.scale
        c.counters, c.sumsq, c.scale = counters, sumsq, scale
        try:
            return {n: c.stats(t, self.weights) for t, n in enumerate(self.names)}
        finally:
            c.counters, c.sumsq, c.scale = saved
