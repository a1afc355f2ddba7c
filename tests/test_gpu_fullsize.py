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
    """Complete neighbour list of every sampled query == the oracle's (the
    ambiguous band counted and recorded for the parity report)."""
    from conftest import record_band
    q_t = torch.from_numpy(qids).to("cuda", torch.int32)
    sel = pairs[torch.isin(pairs[:, 0], q_t)].cpu().numpy().astype(np.int64)
    n_sure = n_amb = n_amb_in = 0
    for qi, (sure, amb) in zip(qids, brute.neighbors_of(D, eps, qids)):
        got = np.sort(sel[sel[:, 0] == qi, 1])
        assert len(np.unique(got)) == len(got), "duplicate neighbour"
        S, G, A = set(sure.tolist()), set(got.tolist()), set(amb.tolist())
        assert S <= G and G <= S | A, (qi, len(S - G), len(G - S - A))
        n_sure, n_amb, n_amb_in = n_sure + len(S), n_amb + len(A), n_amb_in + len(G & A)
    record_band(n_sure, n_amb, n_amb_in)
    return n_amb


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


# Every config point bench.py or DESIGN.md reports (BASELINE.json configs[1..3],
# PAPER.md l.876-877 k sweep, l.968-970 eps ranges), with the flags it runs:
# (workload, eps override, k override, Index flags, sampled queries).
POINTS = [
    ("uniform16", 0.50, None, {}, 24),
    ("uniform16", 0.55, None, {}, 24),
    ("uniform16", 0.60, None, {}, 24),
    ("expo16", None, None, {}, 24),
    ("expo32", None, None, {}, 40),
    ("expo32", None, None, {"reorder": False}, 24),
    ("expo32", None, None, {"sortidu": False}, 24),
    ("songs90", 0.005, 4, {}, 24),
    ("songs90", 0.005, 5, {}, 24),
    ("songs90", 0.005, 6, {}, 24),
    ("songs90", 0.005, 7, {}, 24),
    ("songs90", 0.005, 8, {}, 24),
    ("songs90", 0.01, 6, {}, 16),
]
_DATA = {}


def _data(workload):
    if workload not in _DATA:
        _DATA.clear()
        w = synth.WORKLOADS[workload]
        _DATA[workload] = synth.make(w["gen"], w["count"], w["dims"], seed=0)
    return _DATA[workload]


@pytest.mark.parametrize("workload,eps,k,flags,nq", POINTS,
                         ids=[f"{w}-eps{e}-k{k}-{'-'.join(f'{a}{int(b)}' for a, b in f.items()) or 'default'}"
                              for w, e, k, f, _ in POINTS])
def test_full_size_sampled_and_global(workload, eps, k, flags, nq):
    from paper_1809_09930_b200 import Index
    w = synth.WORKLOADS[workload]
    eps = w["eps"] if eps is None else eps
    k = w["k"] if k is None else k
    D = _data(workload)
    ix = Index(torch.from_numpy(D).cuda(), eps, k, **flags)
    pairs, nb = bench_launch(ix)
    assert nb >= 3
    global_properties(pairs, len(D))
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    ix.self_join_count_async(cnt)
    torch.cuda.synchronize()
    assert int(cnt[0].item()) == pairs.shape[0]
    qids = synth.query_sample(len(D), nq, seed=11)
    sampled_check(D, eps, pairs, qids)
    assert pairs.shape[0] > len(D)
    del pairs, ix
    torch.cuda.empty_cache()


@pytest.mark.parametrize("rank", [7, 1000, 1999])
def test_expo64_10m_entity_partition_share(rank):
    """configs[4] at full size: rank shares of a 2000-way entity partition
    (per-query mode, so every query of the share has its complete neighbour
    list) against the oracle; the heaviest (rank 7: early in the
    heaviest-first order), a middle and the last share."""
    from paper_1809_09930_b200 import Index
    w = synth.WORKLOADS["expo64_10m"]
    D = _data("expo64_10m")
    ix = Index(torch.from_numpy(D).cuda(), w["eps"], w["k"], symmetric=False)
    world = 2000
    pairs, _ = bench_launch(ix, rank, world)
    qs = torch.unique(pairs[:, 0]).cpu().numpy().astype(np.int64)
    assert len(qs) > 100
    qids = np.sort(np.random.default_rng(5 + rank).choice(qs, 12, replace=False))
    sampled_check(D, w["eps"], pairs, qids)
    del pairs, ix
    torch.cuda.empty_cache()
