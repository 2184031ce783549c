"""Shared helpers for the GPU parity tests: run librk on seeded inputs and compare with the oracle."""
import numpy as np

import oracle

TOL_REWARD = 1e-5  # north_star: rewards within 1e-5 relative (expected bit-identical)


def lat_profile(K, B):
    """lat_ns[m][b] = round(f_m * (16.67 ms + 3.333 ms * b)) (PAPER.md:700 anchors)."""
    f = [2.174, 1.679, 1.000] if K == 3 else [1.6 - 0.1 * m for m in range(K)]
    return np.array([[int(round(f[m] * (16.67e6 + 3.333e6 * b))) for b in B] for m in range(K)], np.int64)


def default_cfg(K, B=(16, 32, 64), rates=(64.0, 128.0, 572.0, 1144.0), beta=1.0, tau_ns=560_000_000, queue=False):
    import paper_1804_06087_b200 as rk
    lat = lat_profile(K, B)
    g = rk.RewardCfg(B=list(B), beta=beta, tau_ns=tau_ns, lat_ns=lat, rates=list(rates), want_exceed=True,
                     want_labelled=True, queue=queue)
    o = oracle.RewardCfg(B=list(B), beta=beta, tau_ns=tau_ns, lat_ns=lat, rates=list(rates), want_exceed=True,
                         queue=queue)
    return g, o


def compare_tables(gt: dict, ot, *, K, check_moments=True, exact_avg=False):
    """Votes and counts bit-exact; avg counts exact except oracle-flagged ambiguous pairs."""
    S = (1 << K) - 1
    assert gt["cnt_vote"].shape == (S,)
    np.testing.assert_array_equal(gt["cnt_vote"], ot.cnt_vote, err_msg="vote counts")
    d = np.abs(gt["cnt_avg"].astype(np.int64) - ot.cnt_avg.astype(np.int64))
    amb = ot.n_amb.astype(np.int64)
    assert (d <= amb).all(), f"avg counts differ beyond ambiguous pairs: {np.nonzero(d > amb)[0][:10]}"
    if exact_avg:
        np.testing.assert_array_equal(gt["cnt_avg"], ot.cnt_avg)
    if check_moments and ot.corr is not None:
        np.testing.assert_array_equal(gt["corr"], ot.corr, err_msg="corr")
        np.testing.assert_array_equal(gt["O"], ot.O, err_msg="O")
        np.testing.assert_array_equal(gt["E"], ot.E, err_msg="E")
        np.testing.assert_array_equal(gt["Q"], ot.Q, err_msg="Q")
        for k in ("reward_sur", "reward_lab"):
            a, b = gt[k], getattr(ot, k)
            np.testing.assert_allclose(a, b, rtol=TOL_REWARD, atol=1e-9, err_msg=k)
