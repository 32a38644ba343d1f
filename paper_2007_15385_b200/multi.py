"""Multi-GPU host logic: point shards + the one count all-reduce.

The batch is partitioned into contiguous, `align`-point-aligned ranges (one
per rank). With `align` a multiple of 32, each rank's PIPM mask words start at
word `lo // 32` of the global mask, so per-rank masks concatenate without bit
shifts (the multi-GPU analogue of the reference's thread chunking,
engines.cpp:30-52; masks never depend on the partitioning,
test_engines.cpp:227-241). The only exchanged data is the vector of inside
counts (one u64 per engine), summed with one all-reduce (NCCL on GPUs, gloo in
the CPU tests).
"""
from __future__ import annotations


def shard(m: int, rank: int, world: int, align: int = 1024) -> tuple[int, int]:
    """[lo, hi) of rank `rank`: contiguous, lo a multiple of `align`."""
    if world < 1 or not 0 <= rank < world or align % 32:
        raise ValueError("bad shard request")
    per = -(-m // world)
    per = -(-per // align) * align
    lo = min(m, rank * per)
    return lo, min(m, lo + per)


def reduce_counts(counts, group=None):
    """Sum the per-rank inside counts in place (int64 tensor) across the group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts
