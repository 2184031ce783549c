"""GPU parity of NEXT-1's greedy batching policy (Algorithm 3; reading S1):
rk_greedy_serve against oracle.greedy_serve, every (rate, subset) scenario, integer-exact."""
import numpy as np
import pytest

import oracle
from bench import lat_profile
from test_oracle_reward import gold

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

KEYS = ("served", "overdue", "exceed_ns", "batches", "unserved")


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def ctx_for(rk, K, C=10):
    c = rk.Context(0)
    c.load_ensemble(K, C)
    return c


def compare(g, o):
    for k in KEYS:
        np.testing.assert_array_equal(g[k], o[k], err_msg=k)


def test_worked_example(rk):
    for key in ("S1", "S1b"):
        gd = gold()[key]
        cfg = rk.RewardCfg(B=[2, 4], beta=1.0, tau_ns=1000, lat_ns=np.array([[600, 900]]), rates=[1e7])
        r = ctx_for(rk, 1).greedy_serve(cfg, int(gd["N"]), 50)
        assert r["served"][0, 0] == gd["served"] and r["overdue"][0, 0] == gd["overdue"]
        assert r["exceed_ns"][0, 0] == gd["exceed"] and r["batches"][0, 0] == gd["batches"]
        assert r["unserved"][0, 0] == gd["unserved"]


@pytest.mark.parametrize("K,B,rates,N,delta", [
    (3, [16, 32, 48], [300.0, 3000.0], 700, 0),
    (3, [16, 32, 48], [300.0, 3000.0], 700, 10_000_000),
    (5, [16, 32, 48, 64], [128.0, 572.0], 2000, 56_000_000),   # paper's B, delta = 0.1 tau
    (8, [16, 32, 64, 128, 256], [64.0, 572.0, 1144.0], 5000, 56_000_000),
])
def test_parity_rates(rk, K, B, rates, N, delta):
    lat = lat_profile(K, B)
    g = rk.RewardCfg(B=B, beta=0.5, tau_ns=560_000_000, lat_ns=lat, rates=rates)
    o = oracle.RewardCfg(B=B, beta=0.5, tau_ns=560_000_000, lat_ns=lat, rates=rates)
    acc = np.random.default_rng(K).uniform(0.5, 0.9, (1 << K) - 1)
    r = ctx_for(rk, K).greedy_serve(g, N, delta, acc=acc)
    ro = oracle.greedy_serve(o, K, N, delta)
    compare(r, ro)
    np.testing.assert_array_equal(r["reward"], acc[None, :] * (r["served"].astype(np.float64)
                                                              - 0.5 * r["overdue"].astype(np.float64)))
    assert (ro["overdue"] > 0).any() and (ro["batches"] > 0).all()


def test_parity_caller_arrivals(rk):
    K, B, N = 4, [8, 24], 1500
    arr = np.cumsum(np.random.default_rng(2).integers(0, 3_000_000, N)).astype(np.int64)
    lat = lat_profile(K, B) // 20
    for on_device in (False, True):
        a = torch.from_numpy(arr).cuda() if on_device else arr
        g = rk.RewardCfg(B=B, beta=1.0, tau_ns=40_000_000, lat_ns=lat, arrival_ns=a)
        r = ctx_for(rk, K).greedy_serve(g, N, 2_000_000)
        o = oracle.RewardCfg(B=B, beta=1.0, tau_ns=40_000_000, lat_ns=lat, arrival_ns=arr)
        compare(r, oracle.greedy_serve(o, K, N, 2_000_000))


def test_errors(rk):
    c = ctx_for(rk, 2)
    with pytest.raises(rk.RkError):
        c.greedy_serve(rk.RewardCfg(B=[], beta=1.0, tau_ns=10, lat_ns=np.zeros((2, 0), np.int64), rates=[1.0]), 10, 0)
    with pytest.raises(rk.RkError):
        c.greedy_serve(rk.RewardCfg(B=[4], beta=1.0, tau_ns=10, lat_ns=np.zeros((2, 1), np.int64), rates=[0.0]), 10, 0)


def test_measured_latency_profile(rk):
    """NEXT-1: c(m, b) measured from our own head GEMM + per-request prediction, in integer ns (the
    unit of RewardCfg.lat_ns); positive, and a larger batch never takes less than a third of the time
    of a batch 16x smaller (a loose monotonicity check that survives timer noise)."""
    import torch

    import gen
    from paper_1804_06087_b200.latency import measure_lat_ns

    K, C, D, B = 3, 100, 1024, [16, 256]
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    X = torch.empty((max(B), D), dtype=torch.uint16, device="cuda")
    lab = torch.empty(max(B), dtype=torch.int32, device="cuda")
    gen.dev_labels(1, 0, max(B), C, lab.data_ptr())
    gen.dev_features(1, 0, max(B), D, C, psig, False, X.data_ptr(), lab.data_ptr())
    lat = measure_lat_ns(W, b, sh, B, X, reps=5, warmup=2)
    assert lat.shape == (K, len(B)) and lat.dtype == np.int64
    assert (lat > 0).all() and (lat < 10**9).all()
    assert (lat[:, 1] * 3 >= lat[:, 0]).all()
    cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat, rates=[128.0])  # usable as the profile
    assert cfg.lat_ns.shape == (K, len(B))


# ---- NEXT-1 baseline: asynchronous, one model per batch (reading S2) ----------------------
@pytest.mark.parametrize("K,B,rates,N,delta", [
    (3, [16, 32, 48, 64], [128.0, 572.0, 1144.0], 20_000, 0),          # the paper's trio, r_l / r_u
    (3, [16, 32, 48, 64], [572.0], 20_000, 56_000_000),
    (8, [16, 32, 64, 128, 256], [64.0, 572.0, 2000.0, 5000.0], 50_000, 10_000_000),
])
def test_async_parity(rk, K, B, rates, N, delta):
    lat = lat_profile(K, B)
    g = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat, rates=rates)
    o = oracle.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat, rates=rates)
    acc = np.random.default_rng(K).uniform(0.6, 0.9, K)
    r = ctx_for(rk, K).async_serve(g, N, delta, acc=acc)
    ro = oracle.async_serve(o, K, N, delta, acc=acc)
    for k in KEYS + ("model_batches", "reward"):
        np.testing.assert_array_equal(r[k], ro[k], err_msg=k)


def test_async_hand_worked(rk):
    from test_oracle_async import gold
    g = gold()
    cfg = rk.RewardCfg(B=[2], beta=1.0, tau_ns=250, lat_ns=np.array([[100], [300]]),
                       arrival_ns=np.array(g["A_arrivals"], np.int64))
    r = ctx_for(rk, 2).async_serve(cfg, 6, 0, acc=[0.9, 0.6])
    assert r["overdue"][0] == g["A_overdue"][0] and r["exceed_ns"][0] == g["A_exceed"][0]
    assert r["model_batches"][0].tolist() == [int(x) for x in g["A_model_batches"]]
    assert r["reward"][0] == g["A_reward"][0]


# ---- NEXT-1 serving loop: Algorithm 3 batches of one action through the heads and rk_predict ----------
@pytest.mark.parametrize("K,C,D,v,rate", [(3, 1000, 512, 0b111, 572.0), (3, 1000, 512, 0b100, 272.0),
                                          (5, 100, 256, 0b10110, 2000.0)])
def test_serve_stream(rk, K, C, D, v, rate):
    import gen
    N = 3000
    B = [16, 32, 48, 64]
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = gen.labels(31, 0, N, C)
    X = gen.features(31, 0, N, D, C, psig, False, y=y)
    W = gen.weights(32, K, C, D, f0, df, False)
    b = gen.bias(33, K, C, False)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh)
    lat = lat_profile(K, B)
    cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat, rates=[rate])
    Xd = torch.from_numpy(X).cuda()
    pv = torch.zeros(N, dtype=torch.int32, device="cuda")
    pa = torch.zeros(N, dtype=torch.int32, device="cuda")
    st = ctx.serve_stream(Xd, N, cfg, 56_000_000, v, pv, pa)
    # the policy's counters are those of rk_greedy_serve for (rate, v) ...
    gs = ctx.greedy_serve(cfg, N, 56_000_000)
    for k in KEYS:
        assert st[k] == gs[k][0, v - 1], k
    # ... and every served request carries the prediction of v on its own features (oracle heads + vote /
    # average), unserved ones -1
    ref = oracle.logits_gemm(X, W, b, sh)
    ov, oa = oracle.predict(ref, K, C, v)[:2]
    served = int(st["served"])
    pv, pa = pv.cpu().numpy(), pa.cpu().numpy()
    np.testing.assert_array_equal(pv[:served], ov[:served])
    ap = np.sort(oracle.predict(ref, K, C, v, want_avgprob=True)[2], axis=1)
    clear = (ap[:, -1] - ap[:, -2]) > 1e-5 * ap[:, -1]  # rk_predict averages in fp32 (P2: exact off near-ties)
    m = clear[:served]
    np.testing.assert_array_equal(pa[:served][m], oa[:served][m])
    assert (pv[served:] == -1).all() and (pa[served:] == -1).all()


def test_async_and_stream_errors(rk):
    c = ctx_for(rk, 2)
    lat = np.zeros((2, 1), np.int64)
    with pytest.raises(rk.RkError):  # no batch sizes
        c.async_serve(rk.RewardCfg(B=[], beta=1.0, tau_ns=10, lat_ns=np.zeros((2, 0), np.int64), rates=[1.0]), 10, 0)
    with pytest.raises(rk.RkError):  # non-positive rate
        c.async_serve(rk.RewardCfg(B=[4], beta=1.0, tau_ns=10, lat_ns=lat, rates=[0.0]), 10, 0)
    with pytest.raises(rk.RkError):  # negative latency
        c.async_serve(rk.RewardCfg(B=[4], beta=1.0, tau_ns=10, lat_ns=-lat - 1, rates=[1.0]), 10, 0)
    import gen
    K, C, D, N = 2, 100, 128, 64
    psig, f0, df, sh = gen.head_params(D, C, K)
    X = torch.from_numpy(gen.features(1, 0, N, D, C, psig, False)).cuda()
    h = rk.Context(0)
    h.load_ensemble(K, C, D, torch.from_numpy(gen.weights(2, K, C, D, f0, df, False)).cuda(), None, sh)
    cfg = rk.RewardCfg(B=[16], beta=1.0, tau_ns=10**9, lat_ns=np.zeros((K, 1), np.int64), rates=[100.0])
    pv = torch.zeros(N, dtype=torch.int32, device="cuda")
    with pytest.raises(rk.RkError):  # v = 0 is not an action
        h.serve_stream(X, N, cfg, 0, 0, pv)
    with pytest.raises(rk.RkError):  # two arrival streams
        h.serve_stream(X, N, rk.RewardCfg(B=[16], beta=1.0, tau_ns=10**9, lat_ns=np.zeros((K, 1), np.int64),
                                          rates=[100.0, 200.0]), 0, 1, pv)
    with pytest.raises(rk.RkError):  # host features
        h.serve_stream(X.cpu().numpy(), N, cfg, 0, 1, pv)
    with pytest.raises(rk.RkError):  # a logits-only ensemble has no heads to serve with
        c.serve_stream(X, N, cfg, 0, 1, pv)
