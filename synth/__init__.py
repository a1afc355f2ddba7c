"""Seeded synthetic input generators shared by the oracle tests, the GPU tests
and bench.py.

This module holds NONE of the self-join's arithmetic (no distances, no cells,
no variances): it only draws point sets with the shapes and distributions of
the paper's workloads (§5.1 "Datasets", Table 1) and picks seeded
query samples.  Both sides of every parity test receive the same arrays from
here; neither side imports the other.

Recipes (DESIGN.md §"Input recipe"):

* ``exponential``  -- PAPER.md §5.1 (l.782-783): "synthetic datasets with an
  exponential distribution with lambda=40 ... with coordinates in [0,1]".
  Reading R1: draws > 1 are redrawn (rejection, probability
  e^-40), no min/max renormalisation.  This reading reproduces the paper's
  selectivity ranges (Fig. 5 caption) -- see tests/golden/selectivity_calibration.txt.
* ``uniform``      -- i.i.d. U[0,1) coordinates (BASELINE.json configs[0..1]).
* ``songs_like``   -- |D|=515,345, n=90 (Table 1 "Songs"): clustered points
  (Zipf cluster sizes, heavy-tailed cluster centres, Gaussian spread), min/max
  normalised to [0,1] (§5.1); the first 12 dimensions get the lowest variance
  (§5.4).  Reproduces the paper's Songs selectivity range (see songs_like).
"""
from __future__ import annotations

import numpy as np

__all__ = ["uniform", "exponential", "songs_like", "lattice", "query_sample", "make"]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform(count: int, dims: int, seed: int = 0) -> np.ndarray:
    """|D| x n points, i.i.d. U[0,1), float64, C-contiguous."""
    return np.ascontiguousarray(_rng(seed).random((count, dims)))


def exponential(count: int, dims: int, lam: float = 40.0, seed: int = 0) -> np.ndarray:
    """|D| x n points, i.i.d. Exp(lam) redrawn until <= 1."""
    rng = _rng(seed)
    x = rng.exponential(1.0 / lam, size=(count, dims))
    bad = x > 1.0
    while bad.any():
        x[bad] = rng.exponential(1.0 / lam, size=int(bad.sum()))
        bad = x > 1.0
    return np.ascontiguousarray(x)


def songs_like(count: int = 515_345, dims: int = 90, seed: int = 0, n_clusters: int = 4000,
               sigma: float = 0.005) -> np.ndarray:
    """Songs-shaped synthetic set (Table 1: 515,345 x 90), normalised to [0,1].

    Songs (YearPredictionMSD timbre features) is strongly clustered, which is
    what gives it S_D = 4--1.9k at eps = 0.005--0.01 (Fig. 6b caption, l.936).
    Recipe: n_clusters centres whose dimension j is Student-t(df_j) -- df=1.5
    for the first 12 dims (heavy tails: after min/max normalisation their
    bulk is squeezed into a narrow band, i.e. low variance, §5.4 l.876 "the
    first k<~12 dimensions have low variance"), df rising 3 -> 30 for the other
    78; Zipf(0.8) cluster sizes; each point = its centre + N(0, sigma^2) per
    dim; then x' = (x - min)/(max - min) per dim (§5.1 "We normalize all
    datasets in the range [0,1]").  With the defaults the oracle measures
    S_D ~ 6 at eps 0.005 and ~1.9k at eps 0.01 (30 seeded queries).
    """
    rng = _rng(seed)
    df = np.concatenate([np.full(min(12, dims), 1.5), np.linspace(3.0, 30.0, max(dims - 12, 0))])
    centers = np.empty((n_clusters, dims))
    for j in range(dims):
        centers[:, j] = rng.standard_t(df[j], size=n_clusters)
    w = 1.0 / np.arange(1, n_clusters + 1) ** 0.8
    lab = rng.choice(n_clusters, size=count, p=w / w.sum())
    x = centers[lab] + sigma * rng.standard_normal((count, dims))
    mn, mx = x.min(0), x.max(0)
    span = np.where(mx > mn, mx - mn, 1.0)
    x = (x - mn) / span
    x[:, mx == mn] = 0.0
    return np.ascontiguousarray(x)


def lattice(side: int, dims: int, spacing: float = 1.0) -> np.ndarray:
    """All points of the integer lattice {0..side-1}^n scaled by ``spacing``
    (row-major enumeration).  Used for closed-form neighbour counts."""
    axes = [np.arange(side, dtype=np.float64) * spacing] * dims
    g = np.meshgrid(*axes, indexing="ij")
    return np.ascontiguousarray(np.stack([a.ravel() for a in g], axis=1))


def query_sample(count: int, m: int, seed: int = 1) -> np.ndarray:
    """m distinct query ids in [0, count), sorted, seeded."""
    m = min(m, count)
    return np.sort(_rng(seed).choice(count, size=m, replace=False)).astype(np.int64)


# Named workloads (BASELINE.json "configs"); eps values chosen per DESIGN.md.
WORKLOADS = {
    # configs[0]: N=2000 uniform 16-d, eps for ~8 neighbours/point, k=6
    # (eps=0.96 -> S_D = 8.289, 18,578 ordered pairs, measured with oracle/brute, seed 0)
    "uniform16_small": dict(gen="uniform", count=2000, dims=16, eps=0.96, k=6),
    # configs[1]: N=2M uniform 16-d, k=6, eps sweep 0.50 / 0.55 / 0.60 (S_D ~ 1.1 / 4.7 / 17)
    "uniform16": dict(gen="uniform", count=2_000_000, dims=16, eps=0.55, k=6),
    # Syn16 of Table 1 (Fig. 5a eps range 0.03-0.05)
    "expo16": dict(gen="exponential", count=2_000_000, dims=16, eps=0.04, k=6),
    # configs[2]: N=2M exponential 32-d, k=6 (Syn32 of Table 1; eps range of Fig. 5b)
    "expo32": dict(gen="exponential", count=2_000_000, dims=32, eps=0.08, k=6),
    # configs[3]: Songs-shaped N=515,345 90-d, k sweep 4-8 (Fig. 5/6b eps 0.005-0.01)
    "songs90": dict(gen="songs_like", count=515_345, dims=90, eps=0.005, k=6),
    # configs[4]: N=10M exponential 64-d entity-partitioned (Syn64 eps range)
    "expo64_10m": dict(gen="exponential", count=10_000_000, dims=64, eps=0.16, k=6),
}


def make(gen: str, count: int, dims: int, seed: int = 0, **_) -> np.ndarray:
    if gen == "uniform":
        return uniform(count, dims, seed)
    if gen == "exponential":
        return exponential(count, dims, 40.0, seed)
    if gen == "songs_like":
        return songs_like(count, dims, seed)
    raise ValueError(f"unknown generator {gen!r}")
