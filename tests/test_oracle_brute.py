"""Pins for oracle/brute.py against things other than itself: hand examples,
lattice closed forms, scipy's cKDTree, a 1-D sorted sliding window, and the
trivial limits (§3.1 definition, l.104-110)."""
import math

import numpy as np
import pytest
from scipy.spatial import cKDTree

import synth
from oracle import brute


def as_set(p):
    return {tuple(map(int, r)) for r in p}


def test_hand_1d_example():
    # 1-D {0.0, 0.1, 0.5}, eps=0.15: 0-1 at 0.1 (within), 1-2 at 0.4, 0-2 at 0.5.
    D = np.array([[0.0], [0.1], [0.5]])
    sure, amb = brute.self_join(D, 0.15)
    assert as_set(sure) == {(0, 0), (0, 1), (1, 0), (1, 1), (2, 2)}
    assert len(amb) == 0
    assert brute.selectivity(len(sure), 3) == pytest.approx(2 / 3)


def test_pythagorean_boundary_is_ambiguous_and_inclusive_pairs_listed():
    # (0,0)-(3,4) and (3,4)-(6,8) are at exactly 5: d^2 == eps^2 -> in the band.
    D = np.array([[0.0, 0.0], [3.0, 4.0], [6.0, 8.0]])
    sure, amb = brute.self_join(D, 5.0)
    assert as_set(sure) == {(0, 0), (1, 1), (2, 2)}
    assert as_set(amb) == {(0, 1), (1, 0), (1, 2), (2, 1)}


@pytest.mark.parametrize("side,dims", [(4, 2), (3, 3), (3, 4)])
def test_lattice_closed_forms(side, dims):
    D = synth.lattice(side, dims)
    N = side ** dims
    # eps=1.2: only axis neighbours (distance 1); sqrt(2) > 1.2.
    sure, amb = brute.self_join(D, 1.2)
    assert len(amb) == 0
    assert len(sure) == N + dims * 2 * (side - 1) * side ** (dims - 1)
    # eps=1.5: distance 1 and sqrt(2) (exactly two coords differ by one).
    sure, amb = brute.self_join(D, 1.5)
    expect = (N + dims * 2 * (side - 1) * side ** (dims - 1)
              + math.comb(dims, 2) * (2 * (side - 1)) ** 2 * side ** (dims - 2))
    assert len(amb) == 0 and len(sure) == expect


@pytest.mark.parametrize("dims,count,eps", [(2, 800, 0.05), (5, 700, 0.25), (16, 600, 0.9)])
def test_against_scipy_kdtree(dims, count, eps):
    D = synth.uniform(count, dims, seed=dims)
    sure, amb = brute.self_join(D, eps)
    kd = cKDTree(D).query_pairs(r=eps, output_type="ndarray")
    kd_set = {(int(a), int(b)) for a, b in kd} | {(int(b), int(a)) for a, b in kd}
    kd_set |= {(i, i) for i in range(count)}
    band = as_set(amb)
    assert as_set(sure) - kd_set == set()
    assert (kd_set - as_set(sure)) <= band
    assert len(sure) > count  # non-trivial: some neighbours found


def test_one_dimensional_sliding_window():
    x = synth.uniform(3000, 1, seed=3)[:, 0]
    eps = 0.002
    sure, amb = brute.self_join(x[:, None], eps)
    xs = np.sort(x)
    cnt = np.searchsorted(xs, xs + eps, side="right") - np.searchsorted(xs, xs - eps, side="left")
    assert len(amb) == 0
    assert len(sure) == int(cnt.sum())


def test_limits_all_pairs_and_self_only():
    D = synth.uniform(300, 4, seed=5)
    sure, amb = brute.self_join(D, 2.0 + 1e-9)          # diameter of [0,1]^4 is 2
    assert len(sure) + len(amb) == 300 * 300
    diff = D[:, None, :] - D[None, :, :]
    gap = np.sqrt((diff ** 2).sum(-1) + np.eye(300) * 10).min()
    sure, amb = brute.self_join(D, gap * 0.5)
    assert as_set(sure) == {(i, i) for i in range(300)} and len(amb) == 0


def test_symmetry_reflexivity_and_duplicates():
    D = synth.exponential(500, 6, seed=7)
    D[10] = D[20]                                       # exact duplicate point
    sure, amb = brute.self_join(D, 0.03)
    s = as_set(sure)
    assert all((j, i) in s for (i, j) in s)
    assert all((i, i) in s for i in range(500))
    assert (10, 20) in s and (20, 10) in s
    assert np.all(np.diff(sure[:, 0]) >= 0)            # lexicographic order


def test_neighbors_of_matches_rows():
    D = synth.exponential(900, 8, seed=11)
    sure, _ = brute.self_join(D, 0.04)
    q = synth.query_sample(900, 25, seed=2)
    for qi, (s, a) in zip(q, brute.neighbors_of(D, 0.04, q, chunk=128)):
        assert list(s) == list(sure[sure[:, 0] == qi][:, 1])
        assert len(a) == 0


def test_selectivity_calibration_golden_supports_reading_r1():
    """tests/golden/selectivity_calibration.txt (written by its generator
    script from oracle/ + synth/ only): under reading R1 the exponential sets
    reproduce the paper's S_D ranges (Fig. 5 caption, l.969), min/max
    renormalised ones give S_D ~ 0.  Re-derives the 16-d eps=0.03 row."""
    import os
    rows = np.loadtxt(os.path.join(os.path.dirname(__file__), "golden", "selectivity_calibration.txt"), ndmin=2)
    paper = {(16, 0.03): 4, (16, 0.05): 1200, (32, 0.08): 31, (32, 0.10): 1400, (64, 0.16): 132, (64, 0.18): 2300}
    for dims, eps, raw, nrm in rows:
        ref = paper[(int(dims), round(eps, 2))]
        assert ref / 2.5 <= raw <= ref * 2.5, (dims, eps, raw, ref)
        assert nrm < 0.1
    D = synth.exponential(2_000_000, 16, seed=0)
    q = synth.query_sample(len(D), 100, seed=1)
    sd = np.mean([len(s) + len(a) - 1 for s, a in brute.neighbors_of(D, 0.03, q)])
    assert abs(sd - rows[0, 2]) < 0.01
