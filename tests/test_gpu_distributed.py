"""Multi-process entity partitioning (§6.2 l.1013) on the GPU, through
paper_1809_09930_b200.distributed (the module bench.py runs):

* NCCL at world size 1 -- the NCCL branch of Comm (broadcast, all-reduce,
  barrier) really executes, and the step's pairs equal the oracle's;
* two gloo ranks sharing one GPU -- each rank joins its share of the
  heaviest-first tile order; the shares are disjoint and their union is the
  oracle's self-join; the all-reduced count equals the union's size;
* bench.py itself under torchrun with 2 gloo ranks: its pair total equals the
  oracle's count.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from oracle import brute

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_WORKER = r"""
import os, sys, json, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import synth
from paper_1809_09930_b200.distributed import Comm, EntityPartitionedJoin
backend, out_stem = sys.argv[2], sys.argv[3]
torch.cuda.set_device(0)
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
else:
    dist.init_process_group("gloo")
comm = Comm(device=torch.device("cuda", 0))
D = torch.empty((3000, 16), dtype=torch.float64, device="cuda")
if comm.rank == 0:
    D.copy_(torch.from_numpy(synth.exponential(3000, 16, seed=31)))
out = torch.empty((400000, 2), dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
job = EntityPartitionedJoin(comm, D, 0.045, 6, out, cnt, symmetric=True)
ix, nb, total = job.step()
torch.cuda.synchronize()
n = int(cnt.item())
np.save(f"{out_stem}_rank{comm.rank}.npy", out[:n].cpu().numpy())
json.dump({"rank": comm.rank, "world": comm.world, "backend": comm.backend, "n": n, "total": int(total.item()),
           "n_batches": nb}, open(f"{out_stem}_rank{comm.rank}.json", "w"))
dist.barrier()
dist.destroy_process_group()
"""


def _run(world, backend, tmp_path):
    port = _port()
    stem = str(tmp_path / "share")
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", _WORKER, ROOT, backend, stem], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    for p in procs:
        o, _ = p.communicate(timeout=600)
        assert p.returncode == 0, o[-3000:]
    metas = [json.load(open(f"{stem}_rank{r}.json")) for r in range(world)]
    shares = [np.load(f"{stem}_rank{r}.npy").view(np.uint32).astype(np.int64) for r in range(world)]
    return metas, shares


def _oracle():
    D = synth.exponential(3000, 16, seed=31)
    sure, amb = brute.self_join(D, 0.045)
    assert len(amb) == 0
    return {tuple(r) for r in sure.tolist()}


def test_nccl_world1_step_equals_oracle(tmp_path):
    metas, shares = _run(1, "nccl", tmp_path)
    assert metas[0]["backend"] == "nccl" and metas[0]["world"] == 1
    got = {tuple(r) for r in shares[0].tolist()}
    assert len(got) == len(shares[0]) and got == _oracle()
    assert metas[0]["total"] == len(got)


def test_two_gloo_ranks_union_equals_oracle(tmp_path):
    metas, shares = _run(2, "gloo", tmp_path)
    sets = [{tuple(r) for r in s.tolist()} for s in shares]
    assert all(len(s) == len(a) for s, a in zip(sets, shares))          # no duplicates within a share
    assert not (sets[0] & sets[1])                                       # disjoint shares
    assert sets[0] | sets[1] == _oracle()                                # union = the self-join
    assert all(m["total"] == len(sets[0]) + len(sets[1]) for m in metas)  # all-reduced count
    assert len(sets[0]) > 0 and len(sets[1]) > 0


def test_bench_two_gloo_ranks_pairs_equal_oracle():
    port = _port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--workload", "uniform16_small", "--dist-backend", "gloo",
           "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    w = synth.WORKLOADS["uniform16_small"]
    D = synth.make(w["gen"], w["count"], w["dims"], seed=0)
    sure, amb = brute.self_join(D, w["eps"])
    assert len(sure) <= line["pairs"] <= len(sure) + len(amb)
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "entity-partitioned dp2"
