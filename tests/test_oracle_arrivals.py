"""Pins of the oracle's sine-plus-noise arrival process (NEXT-4, eqs. eq:r1/eq:r2;
reading Q16) against a hand-worked example, the paper's two constraints and the
statistics of the noise -- not against a retyping of the oracle's formula."""
import math
import os

import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "q16_sine_arrivals.txt")


def gold():
    d = {}
    for ln in open(GOLD):
        if ln.startswith("#") or not ln.strip():
            continue
        k, *v = ln.split()
        d[k] = [float(x) for x in v]
    return d


def test_hand_worked_example():
    g = gold()
    k, b = oracle.sine_params(272.0)
    assert abs(k - g["k"][0]) < 5e-3 and abs(b - g["b"][0]) < 5e-3
    T, dl = 4_000_000_000, 1_000_000_000
    assert [oracle.sine_count(272.0, T, dl, 0.0, 0, j) for j in range(4)] == [int(x) for x in g["counts"]]
    a = oracle.sine_arrivals(272.0, T, dl, 0.0, 0, 0, 170)
    assert a[0] == 0 and a[1] == g["t1"][0] and a[156] == g["t156"][0]
    assert a[157] == g["t157"][0] and a[158] == g["t158"][0]


def test_paper_constraints():
    """eq:r2: peak k + b = 1.1 ref; eq:r1: the noiseless rate exceeds ref for 20 % of each period."""
    for ref in (128.0, 272.0, 572.0):
        k, b = oracle.sine_params(ref)
        assert math.isclose(k + b, 1.1 * ref, rel_tol=1e-14)
        th = (np.arange(2_000_000) + 0.5) / 2_000_000 * 2 * np.pi
        frac = np.mean(k * np.sin(th) + b > ref)
        assert abs(frac - 0.2) < 2e-6, frac
        assert b - k > 0  # the noiseless rate never reaches zero


def test_mean_rate_and_noise():
    """Over whole periods the sine integrates to zero: the noiseless count is b * duration within the
    rounding (<= 1/2 per invocation); with noise, the relative deviations phi have mean 0 and std 0.1
    ("phi ~ N(0, 0.1)", read as the standard deviation)."""
    ref, T, dl = 572.0, 400_000_000_000, 1_000_000_000  # 400 invocations per period, >= 30 requests each
    k, b = oracle.sine_params(ref)
    J = 4 * 400
    n0 = sum(oracle.sine_count(ref, T, dl, 0.0, 3, j) for j in range(J))
    assert abs(n0 - b * J * dl / 1e9) <= 0.5 * J
    exact = np.array([dl / 1e9 * (k * math.sin(2 * math.pi * ((j * dl) % T) / T) + b) for j in range(J)])
    n = np.array([oracle.sine_count(ref, T, dl, 0.1, 3, j) for j in range(J)])
    phi = n / exact - 1.0  # plus the rounding: at most 0.5 / 30 relative here
    assert abs(phi.mean()) < 4 * 0.1 / math.sqrt(J) + 2e-3
    assert abs(phi.std() - 0.1) < 0.01


def test_slices_and_order():
    ref, T, dl = 128.0, 500 * 560_000_000, 100_000_000
    full = oracle.sine_arrivals(ref, T, dl, 0.1, 11, 0, 20_000)
    assert np.all(np.diff(full) >= 0)
    np.testing.assert_array_equal(oracle.sine_arrivals(ref, T, dl, 0.1, 11, 7_000, 3_000), full[7_000:10_000])
