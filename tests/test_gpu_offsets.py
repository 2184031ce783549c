"""A4 exactness for large-magnitude logits.

The averaging fast path forms p[m][c] = exp((l - rmax_m) - lsum_m) in fp32 with lsum_m the log-sum
RELATIVE to the row max (rk.h rk_outputs), so its error does not grow with the logits' offset; decisions
whose fp32 relative gap lies inside the band are redone in fp64 as exp(l - max) / sum (the oracle's
order of operations, oracle.c `or_softmax`). Softmax is shift-invariant (PAPER.md:72 averages the
models' softmax outputs), so per-(sample, model) offsets of +-1e3 .. +-1e4 must leave cnt_avg within the
oracle's ambiguous pairs, through rk_score_logits (caller logits) and rk_score (GEMM bias offsets).
"""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import compare_tables, default_cfg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

OFFSETS = (1000.0, -3000.0, 10000.0, -700.0, 3000.0, -10000.0, 2500.0, -1500.0)


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(rk, L, y, K, C, cfg=None, tie=0):
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, tie=tie)
    dl = dev(L)
    ctx.score_logits(dl, L.shape[2], L.shape[0])
    t = ctx.subset_stats(dev(y), cfg)
    torch.cuda.synchronize()
    return t


def near_tie_logits(N, K, C, seed, offsets):
    """Models 0 and 1 nearly tie classes 0 and 1 in their average: l0 = (a, 0, ...), l1 = (0, a + d, ...)
    with d ~ N(0, 3e-4), so the pair's relative avg gap straddles the fp32 band (2e-5); other models and
    classes are background. Then per-model offsets, rounded once to fp32 (the values both sides read)."""
    rng = np.random.default_rng(seed)
    ldc = (C + 3) // 4 * 4
    L = rng.normal(-3.0, 0.7, size=(N, K, ldc))
    a = rng.uniform(0.5, 2.0, N)
    L[:, 0, 0], L[:, 0, 1] = a, 0.0
    L[:, 1, 0], L[:, 1, 1] = 0.0, a + rng.normal(0.0, 3e-4, N)
    L += np.resize(np.asarray(offsets, np.float64), K)[None, :, None]
    L[:, :, C:] = np.nan
    y = rng.integers(0, 2, N).astype(np.int32)
    return L.astype(np.float32), y


@pytest.mark.parametrize("K,C,N", [(2, 3, 200_000), (3, 10, 50_000), (8, 1000, 3000), (10, 300, 800),
                                   (12, 100, 2000), (12, 1000, 200)])
def test_near_ties_with_offsets(rk, K, C, N):
    L, y = near_tie_logits(N, K, C, 100 + K, OFFSETS)
    t = run(rk, L, y, K, C)
    o = oracle.table(L, y, K, C)
    compare_tables(t, o, K=K, check_moments=False)
    # the case is exercised: pairs decided near the band edge went through the fp64 path
    assert t["n_recheck"].sum() > 0


@pytest.mark.parametrize("K,C,N", [(3, 10, 3000), (8, 1000, 1500), (12, 100, 1200), (11, 1000, 150),
                                   (10, 300, 400)])
@pytest.mark.parametrize("scale", [1e3, 1e4])
def test_workload_logits_with_offsets(rk, K, C, N, scale):
    """The calibrated workload (gen.logits) shifted per (sample, model) by +-scale: same tables as the
    oracle on the shifted fp32 values (every path: K <= 8 warp kernels; K >= 9 warp / CTA / batch kernels)."""
    y = gen.labels(K + 50, 0, N, C)
    L = gen.logits(K + 50, 0, N, K, C, y=y).astype(np.float64)
    sh = np.random.default_rng(K).choice([-1.0, 1.0], size=(N, K)) * scale * np.random.default_rng(K + 1).uniform(
        0.5, 1.0, size=(N, K))
    L = (L + sh[:, :, None]).astype(np.float32)
    gcfg, ocfg = default_cfg(K)
    for tie in (0, 1):
        t = run(rk, L, y, K, C, cfg=gcfg, tie=tie)
        o = oracle.table(L, y, K, C, tie=tie, cfg=ocfg)
        compare_tables(t, o, K=K)


@pytest.mark.parametrize("K,C,D,N", [(3, 1000, 512, 600), (8, 1000, 256, 400), (12, 100, 256, 500)])
def test_gemm_bias_offsets(rk, K, C, D, N):
    """rk_score path: integer-mode heads plus per-model bias offsets of +-1e3..1e4 (exact in fp32: the
    logits keep their 1/8 grid), so the GEMM epilogue's rmax / lsum feed the averaging kernels."""
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = gen.labels(77, 0, N, C)
    X = gen.features(77, 0, N, D, C, psig, False, y=y)
    W = gen.weights(78, K, C, D, f0, df, False)
    b = gen.bias(79, K, C, False) + np.asarray(OFFSETS * 2, np.float32)[:K, None]
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh)
    ctx.score(torch.from_numpy(X).cuda(), N)
    gcfg, ocfg = default_cfg(K)
    t = ctx.subset_stats(torch.from_numpy(y).cuda(), gcfg)
    ref = oracle.logits_gemm(X, W, b, sh)
    assert np.abs(ref).max() > 900
    o = oracle.table(ref, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)
