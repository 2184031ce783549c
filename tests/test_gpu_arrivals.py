"""GPU parity of NEXT-4's sine-plus-noise arrival process (eqs. eq:r1/eq:r2; reading Q16):
rk_sine_arrivals against oracle.sine_arrivals, bit-exact (integer ns), including shard slices (n0 > 0),
several invocation intervals and noise levels, and the arrivals feeding the batch moments (A5) and
Algorithm 3 greedy serving (NEXT-1) on the device."""
import numpy as np
import pytest

import gen
import oracle
from bench import lat_profile
from gpu_helpers import compare_tables

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TAU = 560_000_000
PERIOD = 500 * TAU  # PAPER.md:683 "T ... configured to be 500 x tau"


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def gpu_arrivals(rk, ctx, N, ref, period, delta, sigma, seed, n0=0):
    out = torch.empty(max(N, 1), dtype=torch.int64, device="cuda")
    ctx.sine_arrivals(out, N, ref, period, delta, sigma, seed, n0)
    torch.cuda.synchronize()
    return out[:N].cpu().numpy()


@pytest.mark.parametrize("ref,delta,sigma,N,n0", [
    (128.0, 100_000_000, 0.1, 300_000, 0),      # r_l of the paper's trio
    (572.0, 50_000_000, 0.1, 300_000, 12_345),  # r_u, a shard starting mid-stream
    (572.0, 1_000_000_000, 0.0, 100_000, 0),    # noiseless
    (272.0, 7_000_000, 0.3, 50_000, 999),       # few requests per invocation (many zero counts)
])
def test_parity(rk, ref, delta, sigma, N, n0):
    ctx = rk.Context(0)
    g = gpu_arrivals(rk, ctx, N, ref, PERIOD, delta, sigma, 42, n0)
    o = oracle.sine_arrivals(ref, PERIOD, delta, sigma, 42, n0, N)
    np.testing.assert_array_equal(g, o)
    assert np.all(np.diff(g) >= 0)


def test_errors(rk):
    ctx = rk.Context(0)
    out = torch.empty(4, dtype=torch.int64, device="cuda")
    for bad in [dict(ref_rate=0.0), dict(period_ns=0), dict(delta_ns=-1), dict(noise_std=-0.1)]:
        kw = dict(ref_rate=100.0, period_ns=PERIOD, delta_ns=10**8, noise_std=0.1)
        kw.update(bad)
        with pytest.raises(rk.RkError):
            ctx.sine_arrivals(out, 4, kw["ref_rate"], kw["period_ns"], kw["delta_ns"], kw["noise_std"])
    with pytest.raises(rk.RkError):  # host output buffer
        ctx.sine_arrivals(np.zeros(4, np.int64), 4, 100.0, PERIOD, 10**8)


def test_moments_and_serving_on_sine_arrivals(rk):
    """The device arrival times drive the overdue / labelled moments (A5) and greedy serving (NEXT-1):
    both equal the oracle's on the same (oracle-generated) arrivals."""
    K, C, N = 6, 100, 24_576
    B = [16, 32, 64]
    ctx = rk.Context(0)
    arr_d = torch.empty(N, dtype=torch.int64, device="cuda")
    ctx.sine_arrivals(arr_d, N, 572.0, PERIOD, 50_000_000, 0.1, 5)
    arr = oracle.sine_arrivals(572.0, PERIOD, 50_000_000, 0.1, 5, 0, N)
    lat = lat_profile(K, B)
    y = gen.labels(8, 0, N, C)
    L = gen.logits(8, 0, N, K, C, y=y)
    ctx.load_ensemble(K, C)
    dl = torch.from_numpy(L).cuda()
    ctx.score_logits(dl, L.shape[2], N)
    g = rk.RewardCfg(B=B, beta=1.0, tau_ns=TAU, lat_ns=lat, arrival_ns=arr_d, want_exceed=True, want_labelled=True)
    t = ctx.subset_stats(torch.from_numpy(y).cuda(), g)
    o = oracle.RewardCfg(B=B, beta=1.0, tau_ns=TAU, lat_ns=lat, arrival_ns=arr, want_exceed=True)
    ot = oracle.table(L, y, K, C, cfg=o)
    compare_tables(t, ot, K=K)
    assert t["O"].sum() > 0  # the peak rate overloads some subsets
    r = ctx.greedy_serve(g, N, 56_000_000)
    ro = oracle.greedy_serve(o, K, N, 56_000_000)
    for k in ("served", "overdue", "exceed_ns", "batches", "unserved"):
        np.testing.assert_array_equal(r[k], ro[k], err_msg=k)


def test_fullsize_stream(rk):
    """c5's 4M requests at r_u in bench.py's launch configuration (one call): bit-exact against the oracle's
    arrival times, non-decreasing, and the mean rate over the whole span within 2 % of b (the sine term
    integrates to ~0 over the covered periods)."""
    N, ref, delta = 4_000_000, 572.0, 50_000_000
    ctx = rk.Context(0)
    g = gpu_arrivals(rk, ctx, N, ref, PERIOD, delta, 0.1, 17)
    o = oracle.sine_arrivals(ref, PERIOD, delta, 0.1, 17, 0, N)
    np.testing.assert_array_equal(g, o)
    assert np.all(np.diff(g) >= 0)
    k, b = oracle.sine_params(ref)
    span_s = g[-1] / 1e9
    periods = span_s / (PERIOD / 1e9)
    assert periods > 10
    assert abs(N / span_s - b) < 0.02 * b, (N / span_s, b)
