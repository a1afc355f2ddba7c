"""Full-size parity (BASELINE.json configs) in the launch configuration
bench.py times: estimator -> n_b = max(3, ceil(est/b_s)) batches of
gj_self_join_async into one HBM buffer.  The oracle cannot join 2e6 points,
so it checks (a) the complete neighbour lists of seeded sampled queries
(oracle/brute.neighbors_of, one query against all points) and (b) properties
that hold at any size: symmetry, reflexivity, no duplicates, count == the
count-only kernel."""
import numpy as np
import pytest

import synth
from oracle import brute

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()


def bench_launch(ix, rank=0, world=1, b_s=0):
    """Exactly bench.py's step after the index build."""
    from paper_1809_09930_b200 import num_batches
    est = ix.estimate(0.01, rank, world)
    nb = num_batches(est, b_s)
    cap = int(ix.estimate(1.0, rank, world) * 1.02) + 65536
    out = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for b in range(nb):
        ix.self_join_async(out, cnt, b, nb, rank, world)
    torch.cuda.synchronize()
    n = int(cnt.item())
    assert n <= cap
    return out[:n], nb


def sampled_check(D, eps, pairs, qids):
    q_t = torch.from_numpy(qids).to("cuda", torch.int32)
    sel = pairs[torch.isin(pairs[:, 0], q_t)].cpu().numpy().astype(np.int64)
    amb_total = 0
    for qi, (sure, amb) in zip(qids, brute.neighbors_of(D, eps, qids)):
        got = np.sort(sel[sel[:, 0] == qi, 1])
        assert len(np.unique(got)) == len(got), "duplicate neighbour"
        S, G, A = set(sure.tolist()), set(got.tolist()), set(amb.tolist())
        assert S <= G and G <= S | A, (qi, len(S - G), len(G - S - A))
        amb_total += len(A)
    return amb_total


def global_properties(pairs, N):
    p = pairs.to(torch.int64)
    key = (p[:, 0] << 32) | p[:, 1]
    rkey = (p[:, 1] << 32) | p[:, 0]
    ks, _ = torch.sort(key)
    rs, _ = torch.sort(rkey)
    assert torch.equal(ks, rs), "pair set not symmetric"
    assert bool((ks[1:] != ks[:-1]).all()), "duplicate pairs"
    selfs = p[p[:, 0] == p[:, 1], 0]
    assert selfs.numel() == N and torch.unique(selfs).numel() == N, "self pairs missing"


@pytest.mark.parametrize("workload,nq", [("expo32", 40), ("uniform16", 24), ("songs90", 24)])
def test_full_size_sampled_and_global(workload, nq):
    from paper_1809_09930_b200 import Index
    w = synth.WORKLOADS[workload]
    D = synth.make(w["gen"], w["count"], w["dims"], seed=0)
    ix = Index(torch.from_numpy(D).cuda(), w["eps"], w["k"])
    pairs, nb = bench_launch(ix)
    assert nb >= 3
    global_properties(pairs, len(D))
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    ix.self_join_count_async(cnt)
    torch.cuda.synchronize()
    assert int(cnt[0].item()) == pairs.shape[0]
    qids = synth.query_sample(len(D), nq, seed=11)
    sampled_check(D, w["eps"], pairs, qids)
    assert pairs.shape[0] > len(D)


def test_expo64_10m_entity_partition_share():
    """configs[4] at full size: one rank's share of a 2000-way entity
    partition (per-query mode, so every query of the share has its complete
    neighbour list) against the oracle."""
    from paper_1809_09930_b200 import Index
    w = synth.WORKLOADS["expo64_10m"]
    D = synth.make(w["gen"], w["count"], w["dims"], seed=0)
    ix = Index(torch.from_numpy(D).cuda(), w["eps"], w["k"], symmetric=False)
    world, rank = 2000, 7
    pairs, _ = bench_launch(ix, rank, world)
    qs = torch.unique(pairs[:, 0]).cpu().numpy().astype(np.int64)
    assert len(qs) > 100
    qids = np.sort(np.random.default_rng(5).choice(qs, 12, replace=False))
    sampled_check(D, w["eps"], pairs, qids)
