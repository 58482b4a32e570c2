"""Multi-GPU partitioning of the decode hot path.

Two ways to split one box's work, one process per GPU:

* **By sequence** (bench.py's default): each rank owns whole sequences.  Every
  (sequence, layer) unit is independent -- including the layer-scope top-k,
  whose aggregate sums the heads of one sequence's layer (engine.py:317) -- so
  there is no data-path collective.

* **By KV head** (the north star's partitioning): rank r owns kv heads
  [r*Hkv/N, (r+1)*Hkv/N) of every sequence, and their q heads (a GQA group
  stays on one rank).  Its cache holds only those heads: low-bit tier,
  residual window, pinned slots and the pinned-host slow-tier shard.
  - ``topk_scope="kv_head"``: every unit is still local, no exchange.
  - ``topk_scope="layer"`` (reference parity): the speculative row's
    probabilities must be summed over ALL q heads before the top-k.  Each rank
    computes its partial aggregate, the ranks sum them with an all-reduce on the
    cache's copy stream, and every rank then selects the same positions
    (``spc_set_agg_reduce`` / ``spc_agg_buffer`` / ``spc_finish_layer``).  The
    all-reduce sits on the ticket's copy-stream chain, off the attention's
    critical path, like the prefetch it feeds.

The per-rank sums are in ascending local head order and the all-reduce adds
the ranks' partials, so the aggregate differs from the single-GPU one by fp32
reassociation only (~1e-7 relative).  The top-k sets agree except where two
aggregate values are that close (SURVEY 8(c) parity contract (2)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

__all__ = ["HeadShard", "head_shard", "allreduce_sum", "Partition", "plan_partition"]


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_lo: int
    kv_hi: int
    q_lo: int
    q_hi: int

    @property
    def kv_heads(self) -> int:
        return self.kv_hi - self.kv_lo

    @property
    def q_heads(self) -> int:
        return self.q_hi - self.q_lo

    def slice_q(self, x):
        """[..., q_heads_total, d] -> this rank's q heads."""
        return x[..., self.q_lo:self.q_hi, :]

    def slice_kv(self, x):
        """[..., kv_heads_total, d] -> this rank's kv heads."""
        return x[..., self.kv_lo:self.kv_hi, :]


def head_shard(kv_heads: int, q_heads: int, rank: int, world: int) -> HeadShard:
    """Contiguous KV-head ranges, GQA groups kept whole (model.py:47-49:
    q head j reads kv head j // (Hq/Hkv))."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if kv_heads % world:
        raise ValueError(f"kv_heads={kv_heads} does not split over {world} ranks; shard by sequence")
    if q_heads % kv_heads:
        raise ValueError("q_heads must be a multiple of kv_heads")
    per = kv_heads // world
    grp = q_heads // kv_heads
    return HeadShard(rank, world, rank * per, (rank + 1) * per, rank * per * grp, (rank + 1) * per * grp)


def allreduce_sum(group=None):
    """The cross-rank reduction for SpeculativeLayerDecoder(agg_reduce=...):
    an in-place SUM all-reduce over ``group`` (NCCL over NVLink on a GPU box,
    gloo in the CPU-side tests), enqueued on the current stream -- which the
    decoder sets to the cache's copy stream."""
    import torch.distributed as dist

    def reduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return reduce


@dataclass(frozen=True)
class Partition:
    """One rank's share of a (KV head x sequence) partition of a box.

    The world is laid out as ``head_groups`` x ``batch_groups``: rank r owns
    the head shard ``r % head_groups`` of the sequences in batch slice
    ``r // head_groups``.  The ranks of one batch slice together hold every
    head of those sequences, so the layer-scope aggregate (engine.py:317) is
    reduced over ``agg_group`` only; batch slices never exchange data."""
    rank: int
    world: int
    head_groups: int
    batch_groups: int
    heads: HeadShard
    seq_lo: int
    seq_hi: int

    @property
    def batch(self) -> int:
        return self.seq_hi - self.seq_lo

    @property
    def agg_group(self) -> list:
        """Ranks that share this rank's sequences (the agg all-reduce group)."""
        b = self.rank // self.head_groups
        return [b * self.head_groups + h for h in range(self.head_groups)]

    def all_agg_groups(self) -> list:
        return [[b * self.head_groups + h for h in range(self.head_groups)] for b in range(self.batch_groups)]

    def describe(self) -> str:
        return (f"kv-heads x{self.head_groups} * sequences x{self.batch_groups} "
                f"({self.heads.kv_heads} kv / {self.heads.q_heads} q heads, {self.batch} seqs per rank)")


def plan_partition(kv_heads: int, q_heads: int, batch: int, rank: int, world: int,
                   mode: str = "auto") -> Partition:
    """The north star's partitioning of one box: by KV head
    first, by sequence where heads run out.

    mode "auto"  : head_groups = gcd(world, kv_heads), batch_groups = the rest;
    mode "heads" : all ranks split the heads (kv_heads % world == 0);
    mode "seq"   : all ranks split the sequences (no collective at all).
    Raises ValueError when the batch does not split over the batch groups."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if mode == "auto":
        hg = math.gcd(world, kv_heads)
    elif mode == "heads":
        hg = world
    elif mode == "seq":
        hg = 1
    else:
        raise ValueError("mode must be 'auto', 'heads' or 'seq'")
    if kv_heads % hg:
        raise ValueError(f"kv_heads={kv_heads} does not split over {hg} head groups")
    bg = world // hg
    if bg * hg != world or batch % bg:
        raise ValueError(f"batch={batch} does not split over {bg} sequence groups "
                         f"({world} ranks, {hg} head groups)")
    hs = head_shard(kv_heads, q_heads, rank % hg, hg)
    per = batch // bg
    b = rank // hg
    return Partition(rank, world, hg, bg, hs, b * per, (b + 1) * per)
