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
