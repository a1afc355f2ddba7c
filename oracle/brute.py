"""ORACLE (test infrastructure only) -- brute-force epsilon self-join.

PAPER.md §3.1 (l.104-110): points a, b in D are within epsilon when
dist(a,b) <= eps with dist(a,b) = sqrt(sum_j (a(x_j) - b(x_j))^2); the
self-join result is every tuple (a, b) with that property ("E join_eps E").
l.110: "By comparing all points to each other, the worst-case complexity is
O(|D|^2), which can be simply implemented as a nested loop join".

Reading R3: the square root is monotone, so the test is written
d^2 = sum_j (a_j - b_j)^2 <= eps^2, evaluated in float64 (north_star fixes
FP64).  Reading R4: the result holds ORDERED pairs and includes the self pair
(a, a) -- §5.2 (l.800-802) defines S_D = (|R| - |D|)/|D| "excluding a point
finding itself", so |R| counts self matches.  Reading R5: pairs whose exact
d^2 lies within 1e-12*eps^2 of eps^2 are "ambiguous" (rounding order may
decide them either way) and are returned separately (north_star).

Pinned by tests/test_oracle_brute.py (lattice closed forms, scipy cKDTree,
1-D sliding window, hand examples, trivial limits).
"""
from __future__ import annotations

import numpy as np

AMBIG_REL = 1e-12  # north_star: |d^2 - eps^2| <= 1e-12 * eps^2 is ambiguous


def dist_sq_rows(q: np.ndarray, D: np.ndarray) -> np.ndarray:
    """d^2 between one point q (n,) and every row of D (m, n): sum of squared
    coordinate differences (§3.1), float64."""
    diff = D - q[None, :]
    return np.einsum("ij,ij->i", diff, diff)


def self_join(D: np.ndarray, eps: float, block: int = 256, max_points: int = 60_000):
    """Nested-loop self-join of D (|D| x n, float64).

    Returns (sure, ambiguous): int64 arrays of shape (m, 2) holding ordered
    pairs (i, j), lexicographically sorted.  ``sure`` = pairs with
    d^2 < eps^2 (1 - 1e-12); ``ambiguous`` = pairs with
    |d^2 - eps^2| <= 1e-12 eps^2.  Every other pair is outside epsilon.
    """
    D = np.ascontiguousarray(D, dtype=np.float64)
    N = D.shape[0]
    if N > max_points:
        raise ValueError(f"brute-force oracle guard: |D|={N} > {max_points}")
    e2 = float(eps) * float(eps)
    lo, hi = e2 * (1.0 - AMBIG_REL), e2 * (1.0 + AMBIG_REL)
    sure, amb = [], []
    for i0 in range(0, N, block):
        Q = D[i0:i0 + block]
        diff = Q[:, None, :] - D[None, :, :]          # (b, N, n)
        d2 = np.einsum("ijk,ijk->ij", diff, diff)      # (b, N)
        ii, jj = np.nonzero(d2 < lo)
        sure.append(np.stack([ii + i0, jj], 1))
        ii, jj = np.nonzero((d2 >= lo) & (d2 <= hi))
        amb.append(np.stack([ii + i0, jj], 1))
    sure = np.concatenate(sure).astype(np.int64) if sure else np.zeros((0, 2), np.int64)
    amb = np.concatenate(amb).astype(np.int64) if amb else np.zeros((0, 2), np.int64)
    return _lexsort(sure), _lexsort(amb)


def neighbors_of(D: np.ndarray, eps: float, qids, chunk: int = 1 << 18):
    """Sampled oracle for full-size parity: for each query id in ``qids``
    return (sure_ids, ambiguous_ids), sorted int64 arrays of the points j with
    d^2(q, j) < eps^2(1-1e-12) resp. within the band.  O(|qids| * |D|)."""
    D = np.asarray(D, dtype=np.float64)
    e2 = float(eps) * float(eps)
    lo, hi = e2 * (1.0 - AMBIG_REL), e2 * (1.0 + AMBIG_REL)
    out = []
    for q in qids:
        s_parts, a_parts = [], []
        for j0 in range(0, D.shape[0], chunk):
            d2 = dist_sq_rows(D[q], D[j0:j0 + chunk])
            s_parts.append(np.nonzero(d2 < lo)[0] + j0)
            a_parts.append(np.nonzero((d2 >= lo) & (d2 <= hi))[0] + j0)
        out.append((np.concatenate(s_parts).astype(np.int64), np.concatenate(a_parts).astype(np.int64)))
    return out


def selectivity(result_size: int, n_points: int) -> float:
    """PAPER.md §5.2 eq. (l.800): S_D = (|R| - |D|) / |D|."""
    return (result_size - n_points) / n_points


def _lexsort(p: np.ndarray) -> np.ndarray:
    if p.shape[0] == 0:
        return p.reshape(0, 2)
    o = np.lexsort((p[:, 1], p[:, 0]))
    return p[o]
