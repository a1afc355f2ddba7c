"""Multi-GPU entity partitioning (§6.2, l.1008-1037) over
torch.distributed: one process per GPU, NCCL over NVLink for the plumbing.

  1. replicate D from rank 0 with one broadcast ("we store the entire
     dataset on each p_k once", l.1013);
  2. every rank builds the identical index (deterministic kernels);
  3. rank r joins its query tiles Q_l, l = r mod |p| (round robin over the
     heaviest-first tile order, gj_partition) against the full D;
  4. the global pair count is one all-reduce.

The join needs no other exchange: D is replicated, each rank's output pairs
are disjoint and their union is the full self-join.
"""
from __future__ import annotations

import numpy as np

from . import gpujoin


def share_positions(n_tiles: int, rank: int, world: int, batch: int = 0, n_batches: int = 1) -> np.ndarray:
    """Tile positions processed by (rank, batch) -- from the library's own
    gj_partition arithmetic (host only, no GPU needed)."""
    f, s, c = gpujoin.partition(n_tiles, rank, world, batch, n_batches)
    return f + s * np.arange(c, dtype=np.int64)


def replicate(points, src: int = 0, group=None):
    """Broadcast the point tensor from ``src`` to every rank, in place."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(points, src=src, group=group)
    return points


def global_count(local, group=None):
    """All-reduce (sum) of a count tensor, in place."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(local, group=group)
    return local


def entity_partitioned_join(points, eps: float, k: int, out_pairs, count, n_batches: int = 1, group=None,
                            **flags):
    """Steps 1-4 on the calling rank's current CUDA device.  ``points`` is a
    |D| x n float64 CUDA tensor (valid on rank 0, overwritten elsewhere),
    ``out_pairs`` a [cap, 2] int32 CUDA tensor, ``count`` a 1-element int64
    CUDA tensor (zeroed here).  Returns (index, global pair count tensor)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    replicate(points, 0, group)
    ix = gpujoin.Index(points, eps, k, stream=torch.cuda.current_stream().cuda_stream, **flags)
    count.zero_()
    for b in range(n_batches):
        ix.self_join_async(out_pairs, count, b, n_batches, rank, world)
    total = global_count(count.clone(), group)
    return ix, total
