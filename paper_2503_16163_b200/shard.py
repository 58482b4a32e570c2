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

from dataclasses import dataclass

__all__ = ["HeadShard", "head_shard", "allreduce_sum"]


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
