"""Data-parallel multi-GPU driver: one process per GPU, torch.distributed for plumbing.

Decomposition: every rank holds the whole (replicated) graph and
runs the cheap fragment passes; the expensive enumeration passes (pair tables, hub-local
4-cycles, 5-cycles, 5-cliques, 4-clique sums) are split by work unit across ranks
(``shard_index = rank``, ``num_shards = world``).  Every sharded quantity enters the
orbit equations linearly, so each rank's partial n x 73 matrix is exact and the element-
wise sum modulo 2^64 over ranks is the full result bit for bit.  The one exchange step
is that sum: a single NCCL reduce (SUM) of the partial matrices over NVLink.  uint64 sums
are carried in int64 tensors: two's-complement addition wraps exactly like uint64.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import evoke_orbits_edges, NUM_ORBITS


def reduce_partials(partial: torch.Tensor, dst: int = 0, group=None, all_ranks: bool = False) -> torch.Tensor:
    """Sum int64 partial matrices of all ranks (mod 2^64) into rank ``dst`` (or all ranks)."""
    assert partial.dtype == torch.int64
    if all_ranks:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return partial


def orbits_data_parallel(n: int, edges: torch.Tensor, group=None, dst: int = 0, induced: bool = True,
                         stream=None) -> torch.Tensor:
    """Full n x 73 orbit matrix on rank ``dst`` (int64 tensor holding uint64 bits).

    ``edges`` must be a CUDA int32 [m, 2] tensor on this rank's device (replicated input).
    Other ranks return their partial matrix."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    out = torch.empty((n, NUM_ORBITS), dtype=torch.int64, device=edges.device)
    evoke_orbits_edges(n, edges, out=out, induced=induced, shard_index=rank, num_shards=world, stream=stream)
    if world > 1:
        reduce_partials(out, dst=dst, group=group)
    return out
