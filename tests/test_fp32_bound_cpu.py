"""CPU check of the certified FP32 prefilter bound (gj_fp32_threshold;
DESIGN.md §"FP32 prefilter"): the kernel's float32 arithmetic is emulated
exactly (correctly rounded float32 conversions, adds and FMAs via exact
rationals) on adversarial pairs whose exact distance is at or just inside
eps; none may have a float32 running sum above the threshold, at any prefix.
Also checks the threshold stays within a small relative margin of eps^2."""
from fractions import Fraction

import numpy as np
import pytest

from paper_1809_09930_b200 import gpujoin


def f32(fr: Fraction) -> Fraction:
    """Correctly rounded (nearest, ties to even) float32 of an exact rational."""
    x = np.float32(float(fr))
    best = None
    for c in (np.nextafter(x, np.float32(-np.inf)), x, np.nextafter(x, np.float32(np.inf))):
        d = abs(Fraction(float(c)) - fr)
        key = (d, int(np.frombuffer(np.float32(c).tobytes(), np.uint32)[0]) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return Fraction(float(best[1]))


def kernel_sums(q, c, mins):
    """Running float32 sums exactly as k_join32 computes them."""
    a = Fraction(0)
    out = []
    for j in range(len(q)):
        qj = f32(Fraction(float(np.float64(q[j]) - np.float64(mins[j]))))    # fl32(fl64(q - min))
        cj = f32(Fraction(float(np.float64(c[j]) - np.float64(mins[j]))))
        t = f32(qj - cj)                                                   # FADD2 (q + (-c))
        a = f32(t * t + a)                                                 # FFMA2, one rounding
        out.append(a)
    return out


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()


@pytest.mark.parametrize("n,eps,span,shift", [(8, 0.05, 1.0, 0.0), (16, 0.3, 2.0, -1.0), (32, 0.08, 1.0, 0.0),
                                              (24, 1e-2, 1.0, 1000.0), (24, 1e-3, 1.0, 1000.0)])
def test_no_inside_pair_is_rejected(n, eps, span, shift):
    rng = np.random.default_rng(n)
    mins = np.full(n, shift)
    enabled, thr, margin = gpujoin.fp32_threshold(eps, np.full(n, span))
    assert margin > 0
    if not enabled:
        assert margin > 1e-3
        pytest.skip("filter disabled for this spread")
    thr = Fraction(float(thr))
    for _ in range(300):
        q = shift + rng.random(n) * span
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        r = eps * (1 - rng.random() * 1e-7)                  # exact distance at/just inside eps
        c = q + v * r
        c = np.clip(c, shift, shift + span)
        d2 = sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(q, c))
        if d2 > Fraction(eps) ** 2:
            continue
        for s in kernel_sums(q, c, mins):
            assert s <= thr


@pytest.mark.parametrize("n,eps,span,shift", [(8, 0.05, 1.0, 0.0), (32, 0.08, 1.0, 0.0), (90, 0.01, 1.0, 0.0),
                                              (24, 1e-2, 1.0, 1000.0)])
def test_no_outside_pair_is_accepted_without_fp64(n, eps, span, shift):
    """gj_fp32_accept_threshold: a pair whose exact distance is at or beyond
    eps (1 - 1e-9) never has a float32 sum <= thr_in (it must go to the FP64
    test); pairs well inside are accepted (the threshold is useful)."""
    rng = np.random.default_rng(n + 7)
    mins = np.full(n, shift)
    thr_in = gpujoin.fp32_accept_threshold(eps, np.full(n, span))
    enabled, thr, _ = gpujoin.fp32_threshold(eps, np.full(n, span))
    if not enabled:
        pytest.skip("filter disabled for this spread")
    assert 0 < float(thr_in) < eps * eps < float(thr)
    T = Fraction(float(thr_in))
    lim = Fraction(eps) * (1 - Fraction(1, 10 ** 9))
    n_inside_ok = 0
    for i in range(240):
        q = shift + rng.random(n) * span
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        rel = [1 - 5e-10, 1.0, 1 + 1e-7, 0.999][i % 4]       # at / beyond the certain-inside limit, and well inside
        c = np.clip(q + v * eps * rel, shift, shift + span)
        d2 = sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(q, c))
        final = kernel_sums(q, c, mins)[-1]
        if d2 >= lim * lim:
            assert final > T, "an outside / boundary pair would skip the FP64 test"
        elif d2 <= (Fraction(eps) * Fraction(999, 1000)) ** 2 * Fraction(1001, 1000):
            n_inside_ok += final <= T
    assert n_inside_ok > 30


def test_threshold_margin_and_switch_off():
    on, thr, margin = gpujoin.fp32_threshold(0.08, np.full(32, 0.4))
    assert on and 0 < margin < 1e-4 and float(thr) >= 0.08 ** 2
    off, _, _ = gpujoin.fp32_threshold(1e-6, np.full(32, 1e3))     # A > 1e-3 eps -> disabled
    assert not off


@pytest.mark.parametrize("n,eps,span", [(16, 0.05, 1.0), (16, 0.55, 1.0), (32, 0.08, 0.5), (64, 0.16, 1.0),
                                        (90, 0.01, 1.0)])
def test_tensor_core_bound_keeps_inside_pairs(n, eps, span):
    """gj_tc_threshold: for pairs whose exact distance is at/just inside eps,
    exact rounding of the operands to fp16 (as k_make16 does) leaves
    (T - ||q^ - c^||^2) / 2 above the documented worst-case accumulation
    error, so such a pair can never be rejected by the sign test."""
    rng = np.random.default_rng(n)
    S = 2.0 ** np.floor(np.log2(180.0 / max(np.sqrt(n) * span, eps)))
    K = (n + 4 + 15) // 16 * 16
    worst = None
    pairs = []
    for _ in range(200):
        q = rng.random(n) * span
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        c = np.clip(q + v * eps * (1 - rng.random() * 1e-7), 0, span)
        if np.sum((q - c) ** 2) <= eps * eps:
            pairs.append((q, c))
    qh = [np.float16(S * q).astype(np.float64) for q, _ in pairs]
    ch = [np.float16(S * c).astype(np.float64) for _, c in pairs]
    R2 = max(max(np.dot(a, a) for a in qh), max(np.dot(b, b) for b in ch))
    ok, T, margin = gpujoin.tc_threshold(eps, n, K, S, R2)
    assert margin > 0
    if not ok:   # the index would fall back to the FP32 / FP64 scan
        assert margin >= 0.25
        pytest.skip("bound not certifiable for this spread")
    kappa = (K + 2) * 2.0 ** -21
    err = kappa * (2.001 * R2 + 0.5005 * T) + 2.0 ** -22 * (T / 2 + R2) + 2.0 ** -23
    for a, b in zip(qh, ch):
        d2 = sum((Fraction(float(x)) - Fraction(float(y))) ** 2 for x, y in zip(a, b))
        slack = (Fraction(T) - d2) / 2 - Fraction(err)
        worst = slack if worst is None else min(worst, slack)
        assert slack > 0
