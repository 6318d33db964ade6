"""Multi-GPU plumbing (torch.distributed): scenario sharding and the one collective of the path.

Scenarios are independent, so N GPUs shard them by global scenario index (each rank draws and evaluates
[rank * n, (rank + 1) * n) -- weak scaling -- with no data-path collective); the only exchange is one
all-reduce of the per-rank aggregate struct (dstack_agg_t: 5 f64 sums followed by u64 counters and
histograms), SUM for every field.  With the NCCL backend this is a ~2.8 KB all-reduce over NVLink.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .dstack import AGG_WORDS

N_F64 = 5   # leading f64 words of dstack_agg_t


def shard(num_global: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of the contiguous global-index shard of `rank` (strong-scaling split)."""
    return num_global * rank // world, num_global * (rank + 1) // world


def allreduce_agg(agg: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of a dstack_agg_t held in an int64 tensor of AGG_WORDS words."""
    assert agg.dtype == torch.int64 and agg.numel() == AGG_WORDS
    dist.all_reduce(agg[:N_F64].view(torch.float64), op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(agg[N_F64:], op=dist.ReduceOp.SUM, group=group)
    return agg
