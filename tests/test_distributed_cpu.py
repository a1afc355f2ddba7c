"""Multi-process (world size 2, gloo, CPU) checks of the entity-partitioning
host logic (§6.2): replication by broadcast, the all-reduced pair
count, and the round-robin tile assignment of gj_partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import grid


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1809_09930_b200 import distributed as D
        comm = D.Comm()
        assert (comm.rank, comm.world, comm.backend) == (rank, world, "gloo")
        pts = torch.arange(24, dtype=torch.float64).reshape(6, 4) if rank == 0 else torch.zeros(6, 4, dtype=torch.float64)
        comm.broadcast(pts)
        cnt = torch.tensor([10 * (rank + 1)], dtype=torch.int64)
        tot = comm.all_reduce(cnt.clone())
        mx = comm.all_reduce(torch.tensor([1.5 * (rank + 1)], dtype=torch.float64), "max")
        comm.barrier()
        mine = D.share_positions(37, rank, world, 0, 1).tolist()
        q.put((rank, pts.sum().item(), int(tot.item()), mine, float(mx.item())))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


def test_two_rank_gloo_replicate_allreduce_partition():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == float(sum(range(24))) for r in res)          # every rank holds D
    assert all(r[2] == 30 for r in res)                              # 10 + 20
    assert all(r[4] == 3.0 for r in res)                             # max over ranks (bench timing)
    allpos = sorted(res[0][3] + res[1][3])
    assert allpos == list(range(37))                                 # disjoint, complete
    B = _block()
    assert res[0][3] == [j for j in range(37) if (j // B) % 2 == 0]  # query sets of B tiles, round robin


def _block():
    from paper_1809_09930_b200 import gpujoin
    return gpujoin.partition(1, 0, 1)[3]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_partition_matches_paper_round_robin(world):
    # §6.2 l.1013: query set Q_l goes to GPU l mod |p| (oracle/grid.py); a
    # query set is B consecutive heaviest-first tiles (reading R12)
    from paper_1809_09930_b200 import distributed as D
    B = _block()
    assert B >= 1
    n_sets = 32
    ref = grid.assign_query_sets(n_sets, world)
    for r in range(world):
        want = [l * B + i for l in ref[r] for i in range(B)]
        assert D.share_positions(n_sets * B, r, world).tolist() == want
        # a partial last set: T = n_sets * B - 3
        T = n_sets * B - 3
        assert D.share_positions(T, r, world).tolist() == [j for j in want if j < T]


@pytest.mark.parametrize("world,nb,T", [(1, 3, 10), (2, 3, 17), (4, 5, 103), (8, 7, 1000)])
def test_batches_times_ranks_cover_every_tile_once(world, nb, T):
    from paper_1809_09930_b200 import distributed as D
    seen = np.concatenate([D.share_positions(T, r, world, b, nb) for r in range(world) for b in range(nb)])
    assert sorted(seen.tolist()) == list(range(T))
