"""GPU parity of NEXT-3, the fused forward + vote (rk_score_labelled; north_star stages A1 + A3/A4,
PAPER.md:152-154, :72, :407): no logits reach HBM for K <= 8 and C > 128 -- the epilogue keeps the row
statistics, the label's logit and the 16 largest logits per (row, model); the vote stage decides every
subset's average from exact values and bounds, and recomputes (GEMM with logits) only the samples whose
bounds leave a subset undecided. The table must equal the oracle's on the same heads (integer mode:
bit-exact logits) and the unfused path's, in both tie modes, with the fallback route exercised."""
import numpy as np
import pytest

import gen
import oracle
from bench import BETA, CONFIGS, TAU_NS, lat_profile
from gpu_helpers import compare_tables, default_cfg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def heads(K, C, D, N, seed, bias_offsets=None):
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = gen.labels(seed, 0, N, C)
    X = gen.features(seed, 0, N, D, C, psig, False, y=y)
    W = gen.weights(seed + 1, K, C, D, f0, df, False)
    b = gen.bias(seed + 2, K, C, False)
    if bias_offsets is not None:
        b = b + np.asarray(bias_offsets, np.float32)[:K, None]
    return y, X, W, b, sh


def run(rk, K, C, D, N, y, X, W, b, sh, cfg, tie, fused):
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh, tie=tie)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    if fused:
        ctx.score_labelled(Xd, yd, N)
    else:
        ctx.score(Xd, N)
    t = ctx.subset_stats(yd, cfg)
    return t, ctx.vote_diag()


@pytest.mark.parametrize("K,C,D,N", [(8, 1000, 256, 3000), (3, 1000, 512, 2500), (6, 300, 256, 4000),
                                     (2, 129, 128, 3000), (8, 1000, 2048, 700)])
@pytest.mark.parametrize("tie", [0, 1])
def test_fused_parity(rk, K, C, D, N, tie):
    y, X, W, b, sh = heads(K, C, D, N, 40 + K)
    gcfg, ocfg = default_cfg(K)
    t, (work, fb, _) = run(rk, K, C, D, N, y, X, W, b, sh, gcfg, tie, True)
    o = oracle.table(oracle.logits_gemm(X, W, b, sh), y, K, C, tie=tie, cfg=ocfg)
    compare_tables(t, o, K=K)
    tu, _ = run(rk, K, C, D, N, y, X, W, b, sh, gcfg, tie, False)
    for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E"):
        np.testing.assert_array_equal(t[k], tu[k], err_msg=k)
    assert work > 0 and fb <= work


def test_fallback_route_taken(rk):
    """Flat rows (a small logit scale) leave subsets undecided by the 16-entry bounds: those samples go
    through the recompute (GEMM with logits + the streaming averaging kernel), and the table is still the
    oracle's."""
    K, C, D, N = 8, 1000, 256, 2000
    y, X, W, b, _ = heads(K, C, D, N, 7)
    sh = -6
    gcfg, ocfg = default_cfg(K)
    t, (work, fb, _) = run(rk, K, C, D, N, y, X, W, b * 0, sh, gcfg, 0, True)
    o = oracle.table(oracle.logits_gemm(X, W, b * 0, sh), y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)
    assert 0 < fb < work, (work, fb)


def test_fused_bias_offsets(rk):
    """Per-model offsets of +-1e3 .. 1e4 (exact on the 1/8 grid): the kept logits and l_y are relative to
    the exact row max, so the bounds stay exact."""
    K, C, D, N = 8, 1000, 256, 1500
    y, X, W, b, sh = heads(K, C, D, N, 11, bias_offsets=[1000.0, -3000.0, 10000.0, -700.0, 3000.0, -10000.0,
                                                          2500.0, -1500.0])
    gcfg, ocfg = default_cfg(K)
    t, _ = run(rk, K, C, D, N, y, X, W, b, sh, gcfg, 0, True)
    o = oracle.table(oracle.logits_gemm(X, W, b, sh), y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)


def test_fused_multiwave_c4(rk):
    """c4's heads (K = 8, C = 1000, D = 2048) at N = 16,384 (7 waves of GEMM work units), bench reward
    configuration, both tie modes: fused table = oracle table, including the per-group vote counts."""
    c = CONFIGS["c4"]
    K, C, D = c["K"], c["C"], c["D"]
    N = 16_384
    lat = lat_profile(K, c["B"])
    g = rk.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat, rates=c["rates"], want_exceed=True,
                     want_labelled=True)
    ocfg = oracle.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat, rates=c["rates"], want_exceed=True)
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    y = gen.labels(9, 0, N, C)
    X = gen.features(9, 0, N, D, C, psig, False, y=y)
    ref = oracle.logits_gemm(X, W, b, sh)
    for tie in (0, 1):
        ctx = rk.Context(0)
        ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh, tie=tie)
        yd = torch.from_numpy(y).cuda()
        ctx.score_labelled(torch.from_numpy(X).cuda(), yd, N)
        t = ctx.subset_stats(yd, g)
        o = oracle.table(ref, y, K, C, tie=tie, cfg=ocfg, want_bits=True)
        compare_tables(t, o, K=K)
        gs, grp = ctx.group_counts()
        np.testing.assert_array_equal(grp, o.vote_ok.reshape(N // 16, 16, -1).sum(axis=1))


def test_fused_contract(rk):
    K, C, D, N = 3, 500, 128, 300
    y, X, W, b, sh = heads(K, C, D, N, 3)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh)
    yd = torch.from_numpy(y).cuda()
    ctx.score_labelled(torch.from_numpy(X).cuda(), yd, N)
    with pytest.raises(rk.RkError):  # no logits were kept
        ctx.predict(1, pred_vote=torch.zeros(N, dtype=torch.int32, device="cuda"))
    with pytest.raises(rk.RkError):  # different labels than the scored ones
        ctx.subset_stats(torch.from_numpy(y.copy()).cuda())
    assert ctx.outputs()["logits"] is None
    # host labels and NULL at accumulate
    ctx.score_labelled(torch.from_numpy(X).cuda(), y, N)
    ctx.subset_reset(None)
    ctx.subset_accumulate(None)
    t = ctx.subset_finalize()
    o = oracle.table(oracle.logits_gemm(X, W, b, sh), y, K, C)
    compare_tables(t, o, K=K, check_moments=False)
    # a label outside [0, C) is reported, as on the logits path
    ybad = y.copy()
    ybad[5] = C
    ctx.score_labelled(torch.from_numpy(X).cuda(), torch.from_numpy(ybad).cuda(), N)
    with pytest.raises(rk.RkError):
        ctx.subset_stats(None)
