"""Pins for oracle/grid.py (Algorithm 1 on the CPU): the values PAPER.md
prints (Fig. 1 cell ids and neighbour set, Fig. 2 variance order, §4.1 loss,
§3.2.2 batch count, §4.3 scan example, §6.2 assignment, §5.6 cost formula),
plus exact agreement with the brute-force definition over k, dimension order
and every REORDER/SORTIDU/SHORTC combination."""
import math
import os

import numpy as np
import pytest

import synth
from oracle import brute, grid
from conftest import GOLDEN


def paper_constants():
    path = os.path.join(GOLDEN, "paper_constants.txt")
    return {l.split()[0]: float(l.split()[1]) for l in open(path) if l.strip() and not l.startswith("#")}


def as_set(p):
    return {tuple(map(int, r)) for r in p}


def fig1_points(golden):
    xy = golden("fig1_points.txt")
    return np.stack([7.0 - xy[:, 1], xy[:, 0]], axis=1)   # dim1 = row from top, dim2 = col


def test_fig1_nonempty_cells_and_adjacent_search(golden):
    D = fig1_points(golden)
    G = grid.construct_index(D, 1.0, 2)
    assert G["widths"] == [7, 7] and G["base"] == [0, 0]
    assert G["cell_ids"] == [2, 8, 14, 18, 23, 24, 32, 34, 36, 47]
    q = 11                                   # (3.6, 3.85) lies in cell 24
    coords = grid.cell_coords(D[q], 1.0, G["base"])
    assert grid.linearize(coords, G["widths"]) == 24
    adj = [G["cell_ids"][c] for c in grid.get_adj_cells(G, coords)]
    assert sorted(adj) == [18, 23, 24, 32]
    assert len(G["order"]) == len(D)        # O(|D|) storage: one entry per point


def test_fig2_reorder_by_variance(golden):
    X = golden("fig2_points.txt") / 2.5
    _, order = grid.reorder_variance(X, frac=1.0)
    order1 = [int(o) + 1 for o in order]
    assert set(order1[:3]) == {5, 3, 6}
    assert order1[3:] == [4, 1, 2]


def test_search_loss_and_cell_counts(golden):
    const = paper_constants()
    assert round(grid.search_loss(5, 3), 3) == const["search_loss_5_3"]
    assert all(grid.search_loss(n, n) == 0 for n in range(2, 11))
    assert 3 ** 6 == const["search_cells_6d"] and 3 ** 2 == const["search_cells_2d"]
    assert grid.compute_num_batches(int(const["batch_threshold"]), int(const["batch_size"])) == 3
    assert grid.compute_num_batches(10 ** 5, 10 ** 8) == 3
    assert grid.compute_num_batches(10 ** 9, 10 ** 8) == 10


def test_sortidu_scan_example():
    u = np.array([0.1, 0.2, 0.3, 0.9])
    assert grid.sortidu_window(u, 0.25, 0.1) == (1, 3)     # scans exactly {0.2, 0.3}
    assert grid.sortidu_window(u, 5.0, 0.1) == (4, 4)
    assert grid.sortidu_window(u, -5.0, 0.1) == (0, 0)


def test_entity_partition():
    a = grid.assign_query_sets(32, 4)
    assert a[0] == list(range(0, 32, 4)) and all(len(v) == 8 for v in a.values())
    assert grid.assign_query_sets(128, 16)[3] == list(range(3, 128, 16))
    with pytest.raises(ValueError):
        grid.assign_query_sets(30, 4)


def test_sortidu_window_ends_exactly_at_eps():
    """§4.3 l.515-517: r is the first candidate with p(u) - r(u) <= eps (so a
    candidate exactly eps below p(u) is inside) and the scan runs while
    s(u) - p(u) <= eps (so a candidate exactly eps above is inside too); the
    first candidate beyond eps on either side is outside.  Exact binary
    fractions, so no rounding decides the ends."""
    u = np.array([0.0, 0.25, 0.5, 0.75, 1.0, 1.25])
    assert grid.sortidu_window(u, 0.75, 0.5) == (1, 6)      # 0.25 is 0.5 below: in; 1.25 0.5 above: in
    assert grid.sortidu_window(u, 0.75, 0.25) == (2, 5)     # ends at 0.5 and 1.0, both exactly eps
    assert grid.sortidu_window(u, 0.5, 0.0) == (2, 3)       # eps = 0: only the equal coordinate
    assert grid.sortidu_window(u, 0.625, 0.125) == (2, 4)   # 0.5 and 0.75 exactly eps away


def _exact_lattice_join(P, eps_int):
    """Integer brute force (Python ints, no rounding): (i, j) with
    sum_j (a_j - b_j)^2 <= eps^2 (§3.1 l.104-106, reading R3)."""
    pts = [tuple(int(v) for v in row) for row in P]
    e2 = eps_int * eps_int
    return {(i, j) for i, a in enumerate(pts) for j, b in enumerate(pts)
            if sum((x - y) ** 2 for x, y in zip(a, b)) <= e2}


@pytest.mark.parametrize("dims,eps_int", [(4, 2), (5, 3)])
def test_grid_join_exact_boundary_lattice(dims, eps_int):
    """Integer lattice points with an integer eps: many pairs lie EXACTLY at
    distance eps, many of them with |p(u) - c(u)| = eps on the SORTIDU dim
    and 0 elsewhere.  The grid join must return exactly the integer
    brute-force set for every k and flag combination -- a '<' for '<=' at
    either SORTIDU end, at the SHORTC test or in the adjacency range fails."""
    rng = np.random.default_rng(dims * 10 + eps_int)
    P = rng.integers(0, 3 * eps_int + 1, size=(260, dims))
    # for every dim d a pair differing by exactly eps in d only: whichever dim
    # REORDER and k make the SORTIDU dim u, the exactly-at-eps window end occurs
    base = np.full((1, dims), 1)
    P = np.unique(np.concatenate([P, base, base + eps_int * np.eye(dims, dtype=np.int64)]), axis=0)
    P = P.astype(np.float64)
    exact = _exact_lattice_join(P, eps_int)
    sure, amb = brute.self_join(P, float(eps_int))
    assert as_set(sure) | as_set(amb) == exact                 # boundary pairs are in the band and inside
    assert len(amb) >= 50                                     # many pairs exactly at eps
    for k in range(1, dims + 1):
        for reorder in (False, True):
            for sortidu in (False, True):
                P_out, _ = grid.gpu_join(P, float(eps_int), k, reorder, sortidu, shortc=True, frac=1.0)
                assert as_set(P_out) == exact, (k, reorder, sortidu)
    # the exactly-at-eps SORTIDU case is present: a pair differing by eps in u only
    Dr, _ = grid.reorder_variance(P, 1.0)
    G = grid.construct_index(Dr, float(eps_int), 1)
    u = G["u"]
    diff = np.abs(Dr[:, None, :] - Dr[None, :, :])
    only_u = (diff[:, :, u] == eps_int) & (np.delete(diff, u, axis=2).sum(axis=2) == 0)
    assert only_u.any()


def test_linearize_roundtrip_is_bijective():
    widths = [3, 5, 4, 2]
    seen = set()
    for c in np.ndindex(*widths):
        seen.add(grid.linearize(c, widths))
    assert seen == set(range(math.prod(widths)))


def test_shortc_identity_and_work():
    rng = np.random.default_rng(0)
    p = rng.random(16)
    C = rng.random((10000, 16))
    w1, d1 = grid.calc_distance_pts(p, C, 0.9, shortc=True)
    w0, d0 = grid.calc_distance_pts(p, C, 0.9, shortc=False)
    assert np.array_equal(w0, w1)
    assert d1.sum() < d0.sum() and np.all(d1 <= d0)
    w, d = grid.calc_distance_pts(np.zeros(4), np.array([[1.0, 0, 0, 0]]), 0.5, True)
    assert not w[0] and d[0] == 1                        # stops after the first dim


CASES = [("uniform", 600, 4, 0.12), ("exponential", 700, 6, 0.035), ("exponential", 500, 10, 0.06),
         ("uniform", 400, 8, 0.45)]


@pytest.mark.parametrize("gen,count,dims,eps", CASES)
def test_grid_join_equals_definition_for_every_k_and_flag(gen, count, dims, eps):
    D = synth.make(gen, count, dims, seed=count + dims)
    sure, amb = brute.self_join(D, eps)
    S, A = as_set(sure), as_set(amb)
    assert len(S) > count                       # the join has real neighbours
    tests = {}
    # all 8 flag combinations for k <= 3; k = n (3^n cells per query) once,
    # only where 3^n stays small for the pure-Python enumeration.
    combos = [(k, r, s, c) for k in sorted({1, 2, min(3, dims)})
              for r in (False, True) for s in (False, True) for c in (False, True)]
    if dims <= 6:
        combos.append((dims, True, True, True))
    for k, reorder, sortidu, shortc in combos:
        P, cnt = grid.gpu_join(D, eps, k, reorder, sortidu, shortc, frac=0.05)
        got = as_set(P)
        assert S <= got and got <= S | A, (k, reorder, sortidu, shortc)
        tests[(k, reorder, sortidu, shortc)] = cnt
    for (k, r, s, c), cnt in tests.items():
        if k > 3:
            continue
        if s:
            assert cnt["tests"] <= tests[(k, r, False, c)]["tests"]
        if c:
            assert cnt["dims"] <= tests[(k, r, s, False)]["dims"]


def test_dimension_order_invariance():
    D = synth.exponential(500, 7, seed=4)
    P0, _ = grid.gpu_join(D, 0.04, 3, reorder=False)
    perm = np.array([6, 2, 0, 5, 1, 4, 3])
    P1, _ = grid.gpu_join(D[:, perm], 0.04, 3, reorder=False)
    assert as_set(P0) == as_set(P1)


def test_sampled_queries_subset():
    D = synth.exponential(600, 6, seed=9)
    full, _ = grid.gpu_join(D, 0.04, 3)
    q = synth.query_sample(600, 40)
    part, _ = grid.gpu_join(D, 0.04, 3, queries=q)
    assert as_set(part) == {p for p in as_set(full) if p[0] in set(q.tolist())}
