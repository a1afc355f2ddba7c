"""Multi-GPU entity partitioning (§6.2, l.1008-1037) over
torch.distributed: one process per GPU, NCCL over NVLink for the plumbing.

One step of the partitioned self-join (``EntityPartitionedJoin.step``):

  1. replicate D from rank 0 with one broadcast ("we store the entire
     dataset on each p_k once", l.1013);
  2. every rank builds the identical index (deterministic kernels: the same
     sorted point order, cells, tiles and heaviest-first tile order);
  3. rank r joins its query tiles, positions j = r mod |p| of the
     heaviest-first tile order (gj_partition; §6.2 "GPU p_k is assigned Q_l
     if l mod |p| = k"), against the full D -- estimator, n_b = max(3,
     ceil(est / b_s)) batches on three streams (§3.2.2, Fig. 4);
  4. the global pair count is one all-reduce.

No other exchange exists: D is replicated, each rank's output pairs are
disjoint and their union is the full self-join (with symmetric evaluation a
pair is emitted, in both orders, by the rank owning the earlier tile).

``Comm`` hides the backend: ``nccl`` moves device tensors over NVLink
directly; ``gloo`` (CPU tests, several ranks sharing one GPU) stages them
through host memory.  bench.py and the gloo tests run the join through this
module.
"""
from __future__ import annotations

import numpy as np

from . import gpujoin


def share_positions(n_tiles: int, rank: int, world: int, batch: int = 0, n_batches: int = 1) -> np.ndarray:
    """Tile positions processed by (rank, batch) -- from the library's own
    gj_partition arithmetic (host only, no GPU needed)."""
    f, s, c, b = gpujoin.partition(n_tiles, rank, world, batch, n_batches)
    m = np.arange(c, dtype=np.int64)
    return (f + s * (m // b)) * b + m % b


class Comm:
    """rank / world of the default process group (1 rank when it is not
    initialised) and the three collectives the partitioned join needs."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.backend = dist.get_backend(group) if self.on else "none"
        self.device = device

    def _staged(self, t):
        # gloo cannot take CUDA tensors: stage through host memory
        return self.backend != "nccl" and t.is_cuda

    def broadcast(self, t, src: int = 0):
        """In place; rank ``src``'s tensor is the value everywhere.  Runs the
        collective whenever a process group exists (world 1 included)."""
        import torch.distributed as dist
        if not self.on:
            return t
        if self._staged(t):
            h = t.cpu()
            dist.broadcast(h, src=src, group=self.group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=src, group=self.group)
        return t

    def all_reduce(self, t, op: str = "sum"):
        """In place; ``op`` = "sum" or "max"."""
        import torch.distributed as dist
        if not self.on:
            return t
        rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
        if self._staged(t):
            h = t.cpu()
            dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=rop, group=self.group)
        return t

    def barrier(self):
        import torch.distributed as dist
        if not self.on:
            return
        if self.backend == "nccl" and self.device is not None:
            dist.barrier(group=self.group, device_ids=[self.device.index])
        else:
            dist.barrier(group=self.group)


class EntityPartitionedJoin:
    """Steps 1-4 on the calling rank's current CUDA device.

    ``points``: |D| x n float64 CUDA tensor (valid on rank 0; overwritten by
    the broadcast elsewhere).  ``out_pairs``: [cap, 2] int32 CUDA tensor for
    this rank's pairs; ``count``: 1-element int64 CUDA tensor.  ``batch_size``
    is b_s (0 = the HBM-sized default, reading R15)."""

    def __init__(self, comm: Comm, points, eps: float, k: int, out_pairs, count, batch_size: int = 0,
                 stream=None, **flags):
        import torch
        self.comm, self.points, self.eps, self.k = comm, points, eps, k
        self.out, self.count, self.batch_size, self.flags = out_pairs, count, batch_size, flags
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.batch_streams = [torch.cuda.Stream() for _ in range(3)]
        self.batch_done = [torch.cuda.Event() for _ in range(3)]

    def step(self, ev_join=None, ev_phase=None, replicate: bool = True):
        """One pass of the hot path.  Returns (index, n_b, global count tensor).
        ev_join = (start, end) CUDA events bracketing the join kernels;
        ev_phase = events recorded after the broadcast, the build and the
        estimate (all on ``self.stream``)."""
        c, s = self.comm, self.stream
        if replicate:
            c.broadcast(self.points)
        if ev_phase:
            ev_phase[0].record(s)
        ix = gpujoin.Index(self.points, self.eps, self.k, stream=s.cuda_stream, **self.flags)
        if ev_phase:
            ev_phase[1].record(s)
        est = ix.estimate(0.01, c.rank, c.world)
        if ev_phase:
            ev_phase[2].record(s)
        nb = gpujoin.num_batches(est, self.batch_size)
        self.count.zero_()
        if ev_join:
            ev_join[0].record(s)
        # Fig. 4: batches on three streams, so one batch's tail overlaps the next
        start = __import__("torch").cuda.Event()
        start.record(s)
        for bs in self.batch_streams:
            bs.wait_event(start)
        for b in range(nb):
            ix.self_join_async(self.out, self.count, b, nb, c.rank, c.world,
                               stream=self.batch_streams[b % 3].cuda_stream)
        for bs, be in zip(self.batch_streams, self.batch_done):
            be.record(bs)
            s.wait_event(be)
        if ev_join:
            ev_join[1].record(s)
        total = c.all_reduce(self.count.clone())
        return ix, nb, total
