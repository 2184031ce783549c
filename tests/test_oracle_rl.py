"""Pins of the NEXT-2 oracle (§2.4, 426-436 §5.2; reading S3): the environment against
a hand-worked episode, the actor-critic gradients against central finite differences of the losses
(independent of the analytic backpropagation), and the closed forms SPEC.md's rl-agent module states."""
import os

import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "s3_env_example.txt")


def gold():
    d = {}
    for ln in open(GOLD):
        if ln.startswith("#") or not ln.strip():
            continue
        k, *v = ln.split()
        d[k] = [float(x) for x in v]
    return d


def test_env_hand_worked():
    g = gold()
    r = oracle.env_rollout(2, [1, 2], [[10, 15], [30, 40]], 50, 1.0, [0.9, 0.6, 0.95],
                           np.array(g["arrivals"], np.int64), 2, [int(a) for a in g["actions"]], 0)
    np.testing.assert_allclose(r["rewards"], g["rewards"], rtol=0, atol=1e-12)
    for k in ("overdue", "t_dec", "t_start", "t_done"):
        assert r[k].tolist() == [int(x) for x in g[k]], k
    for i in range(3):
        np.testing.assert_array_equal(r["states"][i], np.array(g[f"s{i}"], np.float32))


def _problem(seed, F=5, H=4, A=6, E=3, n=4):
    rng = np.random.default_rng(seed)
    P = rng.normal(0, 0.5, oracle.ac_param_count(F, H, A))
    st = rng.normal(0, 1, (E, n, F)).astype(np.float32)
    act = rng.integers(0, A, (E, n)).astype(np.int32)
    rew = rng.uniform(-1, 3, (E, n))
    return F, H, A, P, st, act, rew


import pytest


@pytest.mark.parametrize("ent", [0.0, 0.3])
def test_gradients_match_finite_differences(ent):
    F, H, A, P, st, act, rew = _problem(1)
    g, lp, lv = oracle.ac_grad(F, H, A, P, st, act, rew, 0.9, 0.5, ent)
    npol = H * F + H + A * H + A
    eps = 1e-6
    for i in range(P.size):
        d = np.zeros_like(P)
        d[i] = eps
        _, lp1, lv1 = oracle.ac_grad(F, H, A, P + d, st, act, rew, 0.9, 0.5, ent)
        _, lp0, lv0 = oracle.ac_grad(F, H, A, P - d, st, act, rew, 0.9, 0.5, ent)
        # policy parameters: the policy loss with the advantage held fixed; value parameters: the value loss
        fd = (lp1 - lp0) / (2 * eps) if i < npol else (lv1 - lv0) / (2 * eps)
        if i < npol:  # the advantage depends on value parameters only, so the policy FD is exact to O(eps^2)
            assert abs(fd - g[i]) <= 1e-6 * max(1.0, abs(g[i])), (i, fd, g[i])
        else:
            assert abs(fd - g[i]) <= 1e-6 * max(1.0, abs(g[i])), (i, fd, g[i])


def test_closed_forms():
    F, H, A = 5, 4, 6
    n = 10
    P = np.zeros(oracle.ac_param_count(F, H, A))
    st = np.random.default_rng(2).normal(0, 1, (1, n, F)).astype(np.float32)
    act = np.zeros((1, n), np.int32)
    # zero weights: uniform policy, log pi = -log A; zero value: V = 0
    rew = np.ones((1, n))
    g, lp, lv = oracle.ac_grad(F, H, A, P, st, act, rew, 0.5, 1.0)
    G = 2.0 * (1.0 - 0.5 ** (n - np.arange(n)))  # geometric returns; G_0 = 1.998046875 (SPEC.md rl-agent)
    assert G[0] == 1.998046875
    assert abs(lv - np.mean(G**2)) < 1e-12
    assert abs(lp - np.mean(G) * np.log(A)) < 1e-12
    # zero rewards and zero value: zero advantage -> zero policy gradient
    g, lp, lv = oracle.ac_grad(F, H, A, P, st, act, np.zeros((1, n)), 0.5, 1.0)
    assert np.all(g == 0.0) and lp == 0.0 and lv == 0.0
    # gamma = 0: the return is the (scaled) reward itself
    rew = np.arange(n, dtype=np.float64)[None]
    _, _, lv = oracle.ac_grad(F, H, A, P, st, act, rew, 0.0, 0.25)
    assert abs(lv - np.mean((0.25 * rew) ** 2)) < 1e-12


def test_entropy_term_closed_form():
    """Zero weights: the policy is uniform, H = log A, and with zero advantage the policy loss is -c log A
    and the gradient is zero (the uniform policy is the entropy maximum)."""
    F, H, A = 5, 4, 6
    n = 4
    P = np.zeros(oracle.ac_param_count(F, H, A))
    st = np.random.default_rng(3).normal(0, 1, (1, n, F)).astype(np.float32)
    g, lp, lv = oracle.ac_grad(F, H, A, P, st, np.zeros((1, n), np.int32), np.zeros((1, n)), 0.9, 1.0, 0.5)
    assert abs(lp - (-0.5 * np.log(A))) < 1e-12
    assert np.abs(g).max() < 1e-15
