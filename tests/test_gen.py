"""Generator tests (T1): determinism per seed, slice independence, calibration bands."""
import numpy as np
import pytest

import gen


def test_determinism_and_slices():
    a = gen.logits(7, 0, 300, 4, 37)
    b = gen.logits(7, 0, 300, 4, 37)
    assert np.array_equal(a, b, equal_nan=True)
    s = gen.logits(7, 120, 50, 4, 37)
    assert np.array_equal(a[120:170], s, equal_nan=True)
    assert np.isnan(a[:, :, 37:]).all()  # padding columns are never meaningful
    y = gen.labels(7, 0, 1000, 37)
    assert np.array_equal(gen.labels(7, 400, 100, 37), y[400:500])
    assert y.min() >= 0 and y.max() < 37
    X = gen.features(3, 0, 20, 64, 10, 4000, False)
    assert np.array_equal(gen.features(3, 5, 10, 64, 10, 4000, False), X[5:15])
    vals = gen.bf16_to_f64(X)
    assert set(np.unique(vals)).issubset({-1.0, 0.0, 1.0})


def test_logits_are_dyadic_exact():
    L = gen.logits(1, 0, 50, 3, 100)[:, :, :100]
    # every value is an integer multiple of 2^-24 (exact conversion of the integer numerator)
    assert np.all(np.floor(L.astype(np.float64) * 2**24) == L.astype(np.float64) * 2**24)


@pytest.mark.parametrize("K,C", [(3, 1000), (8, 1000), (12, 100), (3, 10)])
def test_calibration_bands(K, C):
    """Per-model top-1 accuracy in the Inception-like band and correlated errors."""
    N = 1500
    y = gen.labels(11, 0, N, C)
    L = gen.logits(11, 0, N, K, C, y=y)[:, :, :C].astype(np.float64)
    acc = (L.argmax(2) == y[:, None]).mean(0)
    assert acc.min() > 0.60 and acc.max() < 0.92
    top = L.argmax(2)
    unanimous = (top == top[:, :1]).all(1).mean()
    assert 0.3 < unanimous < 0.9
    P = np.exp(L - L.max(2, keepdims=True)); P /= P.sum(2, keepdims=True)
    assert (P.mean(1).argmax(1) == y).mean() >= acc.max()  # averaging does not hurt


def test_head_workload_bands():
    """The bench's c4 heads (gen.head_params, integer mode) sit in SURVEY.md §8(d)'s K = 8 / C = 1000 bands
    (VERDICT r1 weak #8): per-model top-1 in the Inception-like range, ~59% unanimous, mean max-softmax
    0.65-0.80, a candidate set of several classes, and a full-set averaging gain of a few points. Stats in
    fp64 numpy (a workload check, not the method: argmax / softmax are library calls here)."""
    K, C, D, N = 8, 1000, 2048, 1200
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = gen.labels(21, 0, N, C)
    X = gen.bf16_to_f64(gen.features(21, 0, N, D, C, psig, False, y=y)).astype(np.float32)
    W = gen.bf16_to_f64(gen.weights(1000, K, C, D, f0, df, False)).astype(np.float32)
    b = gen.bias(2000, K, C, False).astype(np.float64)
    L = np.einsum("nd,mcd->nmc", X, W, optimize=True).astype(np.float64) * 2.0**sh + b[None]
    top = L.argmax(2)
    acc = (top == y[:, None]).mean(0)
    assert 0.70 < acc.min() and acc.max() < 0.86, acc
    una = (top == top[:, :1]).all(1).mean()
    assert 0.48 < una < 0.66, una
    P = np.exp(L - L.max(2, keepdims=True))
    P /= P.sum(2, keepdims=True)
    assert 0.70 < P.max(2).mean() < 0.82
    theta = P.max(2).min(1) / K
    sc = (P >= theta[:, None, None]).any(1).sum(1).mean()
    assert 5.5 < sc < 11.0, sc
    gain = (P.mean(1).argmax(1) == y).mean() - acc.max()
    assert 0.005 < gain < 0.07, gain


def test_head_workload_bands_c5():
    """c5's heads (K = 12, C = 100, D = 1024) against SURVEY.md §8(d)'s K = 12 row: per-model top-1 in the
    0.68-0.83 range, about half the samples unanimous, mean max-softmax ~0.76, |S_c| ~8."""
    K, C, D, N = 12, 100, 1024, 1500
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = gen.labels(22, 0, N, C)
    X = gen.bf16_to_f64(gen.features(22, 0, N, D, C, psig, False, y=y)).astype(np.float32)
    W = gen.bf16_to_f64(gen.weights(1000, K, C, D, f0, df, False)).astype(np.float32)
    b = gen.bias(2000, K, C, False).astype(np.float64)
    L = np.einsum("nd,mcd->nmc", X, W, optimize=True).astype(np.float64) * 2.0**sh + b[None]
    top = L.argmax(2)
    acc = (top == y[:, None]).mean(0)
    assert 0.68 < acc.min() and acc.max() < 0.85, acc
    una = (top == top[:, :1]).all(1).mean()
    assert 0.42 < una < 0.58, una
    P = np.exp(L - L.max(2, keepdims=True))
    P /= P.sum(2, keepdims=True)
    assert 0.70 < P.max(2).mean() < 0.85
    sc = (P >= (P.max(2).min(1) / K)[:, None, None]).any(1).sum(1).mean()
    assert 5.0 < sc < 10.0, sc
