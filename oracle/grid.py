"""ORACLE (test infrastructure only) -- CPU grid self-join, Algorithm 1 step by step.

Follows PAPER.md in the paper's order and notation; no blocking, fusion or
reordering beyond what the paper states.  Shares no code with oracle/brute.py
or with the CUDA path.  Python loops over queries and cells (small inputs
only); numpy only vectorises the scan over the candidates of one cell.

Citations (PAPER.md line numbers):
  reorderVariance   §4.2 l.498-501   "use a sample of 1% of |D| and estimate
                    the variance in each dimension ... reorder ... from highest
                    to lowest variance"
  constructIndex    §3.2.1 l.121-123 cells of length eps, only non-empty cells,
                    "lookup array that stores the linearized ids of the
                    non-empty grid cells"; §4.1 l.252 index only k of n dims
  getAdjCells       §3.2.1 l.185 "search the adjacent cells (and its origin
                    cell)"; §5.6 l.896 "perform a binary search to find the
                    non-empty cells that exist in the index"
  SORTIDU           §4.3 l.512-520 sort each cell by the un-indexed dim u,
                    binary-search p(u) to r, scan to s
  SHORTC            §4.4 l.555-559 stop once the partial sum exceeds eps
  computeNumBatches §3.2.2 l.199-200 n_b >= 3, b_s
  selectivity       §5.2 l.800
  entity partition  §6.2 l.1013 "GPU p_k is assigned Q_l ... if l mod |p| = k"
  search loss       §4.1 l.252 l(n,k) = (3^n - 3^k)/3^n

Readings (DESIGN.md §"Readings"): R2 grid edges on the eps-lattice through 0
(cell_j = floor(x_j/eps) - floor(min_j/eps)); R6 the 1% variance sample is
every round(1/f)-th point from point 0, unbiased variance, ties -> lower dim
first; R7 u = the (k+1)-th reordered dim when k < n, else dim 1; R8 SHORTC
checks after every dimension; R9 linearisation row-major, first indexed dim
most significant.
"""
from __future__ import annotations

import bisect
import itertools
import math

import numpy as np


# ----------------------------------------------------------------- §4.2 REORDER
def variance_sample_ids(n_points: int, frac: float) -> np.ndarray:
    """R6: every round(1/frac)-th point starting from point 0 (~frac*|D| points)."""
    step = max(1, int(round(1.0 / frac)))
    return np.arange(0, n_points, step, dtype=np.int64)


def estimate_variance(D: np.ndarray, frac: float = 0.01) -> np.ndarray:
    """Per-dimension unbiased sample variance over the 1% sample (§4.2 l.498)."""
    S = D[variance_sample_ids(D.shape[0], frac)]
    m = S.shape[0]
    if m < 2:
        return np.zeros(D.shape[1])
    mean = S.sum(axis=0) / m
    return ((S - mean) ** 2).sum(axis=0) / (m - 1)


def reorder_variance(D: np.ndarray, frac: float = 0.01):
    """§4.2: permute dimensions so variance is non-increasing.  Returns
    (D_reordered, dim_order) with D_reordered[:, t] = D[:, dim_order[t]]."""
    var = estimate_variance(D, frac)
    order = sorted(range(D.shape[1]), key=lambda j: (-var[j], j))   # ties: lower dim first
    order = np.asarray(order, dtype=np.int64)
    return np.ascontiguousarray(D[:, order]), order


# ------------------------------------------------------------ §3.2.1 the grid
def search_loss(n: int, k: int) -> float:
    """§4.1 l.252: l(n,k) = (3^n - 3^k) / 3^n."""
    return (3 ** n - 3 ** k) / 3 ** n


def linearize(coords, widths) -> int:
    """R9: row-major linear id, first indexed dimension most significant."""
    lid = 0
    for c, w in zip(coords, widths):
        lid = lid * int(w) + int(c)
    return lid


def cell_coords(x: np.ndarray, eps: float, base) -> list:
    """R2: c_j = floor(x_j / eps) - base_j for the indexed dims of one point."""
    return [int(math.floor(float(x[t]) / eps)) - int(base[t]) for t in range(len(base))]


def construct_index(Dr: np.ndarray, eps: float, k: int):
    """constructIndex(D, k) (Alg. 1 l.582) over the first k dims of Dr.

    Returns a dict: base, widths, u (sort dim), order (point ids sorted by
    (cell id, u-coordinate)), cell_ids (sorted non-empty linear ids),
    cell_start (|G|+1 offsets into order), cell_of_point.
    """
    N, n = Dr.shape
    if not (1 <= k <= n):
        raise ValueError("need 1 <= k <= n")
    mins, maxs = Dr[:, :k].min(axis=0), Dr[:, :k].max(axis=0)
    base = [int(math.floor(float(m) / eps)) for m in mins]
    widths = [int(math.floor(float(M) / eps)) - b + 1 for M, b in zip(maxs, base)]
    if math.prod(widths) >= 2 ** 63:
        raise OverflowError("linearized cell id overflows 63 bits; choose a smaller k")
    u = k if k < n else 0                       # R7
    lin = [linearize(cell_coords(Dr[i], eps, base), widths) for i in range(N)]
    order = sorted(range(N), key=lambda i: (lin[i], float(Dr[i, u]), i))
    cell_ids, cell_start = [], []
    for pos, i in enumerate(order):
        if not cell_ids or lin[i] != cell_ids[-1]:
            cell_ids.append(lin[i])
            cell_start.append(pos)
    cell_start.append(N)
    return dict(base=base, widths=widths, u=u, k=k, eps=eps, order=np.asarray(order, np.int64),
                cell_ids=cell_ids, cell_start=cell_start, lin=lin)


def get_adj_cells(G, coords):
    """getAdjCells(G, k, point) (Alg. 1 l.600): the up-to-3^k cells adjacent to
    ``coords`` (itself included), offsets enumerated row-major over {-1,0,1}^k,
    each located by binary search in the sorted non-empty id array.  Returns
    the indices (into cell_ids) of the non-empty ones."""
    found = []
    for off in itertools.product((-1, 0, 1), repeat=len(coords)):
        nb = [c + o for c, o in zip(coords, off)]
        if any(c < 0 or c >= w for c, w in zip(nb, G["widths"])):
            continue
        lid = linearize(nb, G["widths"])
        pos = bisect.bisect_left(G["cell_ids"], lid)
        if pos < len(G["cell_ids"]) and G["cell_ids"][pos] == lid:
            found.append(pos)
    return found


# ------------------------------------------------------------- §4.3 / §4.4
def sortidu_window(u_vals: np.ndarray, pu: float, eps: float):
    """§4.3 l.515-517: first candidate r with p(u) - r(u) <= eps (binary
    search), then scan by increasing u until s with s(u) - p(u) > eps.
    Returns the half-open index range [r, s)."""
    lo, hi = 0, len(u_vals)
    while lo < hi:                                    # binary search for r
        mid = (lo + hi) // 2
        if pu - float(u_vals[mid]) <= eps:
            hi = mid
        else:
            lo = mid + 1
    s = lo
    while s < len(u_vals) and float(u_vals[s]) - pu <= eps:   # scan to s
        s += 1
    return lo, s


def calc_distance_pts(p: np.ndarray, C: np.ndarray, eps: float, shortc: bool):
    """calcDistancePts (Alg. 1 l.602) of query p against candidate rows C.

    The partial sum over dims 1..j is accumulated in dimension order; with
    SHORTC the test stops after the first dimension at which the partial sum
    exceeds eps^2 (R8).  Returns (within: bool[m], dims_evaluated: int[m])."""
    n = p.shape[0]
    if C.shape[0] == 0:
        return np.zeros(0, bool), np.zeros(0, np.int64)
    partial = np.cumsum((C - p[None, :]) ** 2, axis=1)    # running sum, dim order
    e2 = eps * eps
    within = partial[:, -1] <= e2
    if not shortc:
        return within, np.full(C.shape[0], n, np.int64)
    over = partial > e2
    first = np.where(over.any(axis=1), over.argmax(axis=1) + 1, n)
    return within, first.astype(np.int64)


# ---------------------------------------------------------------- Algorithm 1
def self_join_kernel(Dr, G, qpos: int, sortidu: bool, shortc: bool, counters: dict):
    """SelfJoinKernel for the query at sorted position ``qpos`` (Alg. 1
    l.596-607).  Returns the sorted positions of its neighbours."""
    eps = G["eps"]
    qid = int(G["order"][qpos])
    p = Dr[qid]
    coords = cell_coords(p, eps, G["base"])
    res = []
    for cidx in get_adj_cells(G, coords):
        a, b = G["cell_start"][cidx], G["cell_start"][cidx + 1]
        counters["cells"] += 1
        if sortidu:
            uvals = Dr[G["order"][a:b], G["u"]]
            r, s = sortidu_window(uvals, float(p[G["u"]]), eps)
            a, b = a + r, a + s
        ids = G["order"][a:b]
        within, dims = calc_distance_pts(p, Dr[ids], eps, shortc)
        counters["tests"] += len(ids)
        counters["dims"] += int(dims.sum())
        res.extend(range(a, b)[i] for i in np.nonzero(within)[0])
    return res


def gpu_join(D: np.ndarray, eps: float, k: int, reorder: bool = True, sortidu: bool = True,
             shortc: bool = True, frac: float = 0.01, queries=None):
    """GPU-Join (Alg. 1 l.579-592) on the CPU.  Returns (pairs, counters):
    pairs = lexicographically sorted int64 (m, 2) ordered pairs of ORIGINAL
    point ids (self pairs included); counters = cells visited, distance tests
    and dimensions evaluated (the SHORTC work counter)."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    if reorder:
        Dr, _ = reorder_variance(D, frac)
    else:
        Dr = D
    G = construct_index(Dr, eps, k)
    counters = dict(cells=0, tests=0, dims=0)
    pos_of = np.empty(D.shape[0], np.int64)
    pos_of[G["order"]] = np.arange(D.shape[0])
    qpositions = range(D.shape[0]) if queries is None else [int(pos_of[q]) for q in queries]
    pairs = []
    for qp in qpositions:
        qi = int(G["order"][qp])
        for np_ in self_join_kernel(Dr, G, qp, sortidu, shortc, counters):
            pairs.append((qi, int(G["order"][np_])))
    P = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if P.shape[0]:
        P = P[np.lexsort((P[:, 1], P[:, 0]))]
    return P, counters


# --------------------------------------------------------- batching (§3.2.2)
def compute_num_batches(est_result: int, batch_size: int, min_batches: int = 3) -> int:
    """§3.2.2 l.199-200: n_b from the estimated |R| and b_s, n_b >= 3."""
    return max(min_batches, -(-int(est_result) // int(batch_size)))


def selectivity(result_size: int, n_points: int) -> float:
    """§5.2 l.800: S_D = (|R| - |D|)/|D|."""
    return (result_size - n_points) / n_points


# ------------------------------------------------ entity partitioning (§6.2)
def assign_query_sets(n_sets: int, n_gpus: int):
    """§6.2 l.1013: query set Q_l goes to GPU p_k iff l mod |p| = k; N_b must
    be a multiple of |p|."""
    if n_sets % n_gpus:
        raise ValueError("N_b mod |p| must be 0")
    return {g: [l for l in range(n_sets) if l % n_gpus == g] for g in range(n_gpus)}
