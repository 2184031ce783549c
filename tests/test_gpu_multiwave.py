"""Whole-table parity at multi-wave sizes of the bench shapes.

The vote-stage kernels keep many samples in flight (the K = 8 averaging kernel alone has ~3k resident
warps), so tables are compared with the oracle at sizes where every kernel runs several grid waves and
its multi-iteration paths are taken:

  * c4 shape: K = 8, C = 1000, N = 131,072, B = {16, ..., 256}, the bench's 4 rates, both tie modes;
  * c5 shape: K = 12, C = 100, N = 65,536, same reward configuration, both tie modes;
  * c4 heads through rk_score (tcgen05 GEMM, integer mode) at N = 16,384 (64 CTA-pair row tiles x 8
    models = 7 waves of work units), both tie modes; this path also runs the averaging kernel's row
    skipping (rows proven by the GEMM's second-largest logit to add only y to the candidate set).

Compared: cnt_vote, corr, O, Q, E bit-exact; cnt_avg within the oracle's ambiguous pairs; rewards within
1e-5; and the per-(16-sample group, subset) vote counts behind Q (rk_group_counts) element by element
against the oracle's per-sample vote bits summed per group -- the per-sample decisions of all S subsets
are checked, not only their totals. Inputs are the seeded workload recipe.
"""
import numpy as np
import pytest

import gen
import oracle
from bench import BETA, CONFIGS, TAU_NS, lat_profile
from gpu_helpers import compare_tables

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def cfgs(rk, name):
    c = CONFIGS[name]
    lat = lat_profile(c["K"], c["B"])
    g = rk.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat, rates=c["rates"], want_exceed=True,
                     want_labelled=True)
    o = oracle.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat, rates=c["rates"], want_exceed=True)
    return c, g, o


def check_groups(ctx, o, N, S):
    gs, grp = ctx.group_counts()
    assert gs == 16 and grp.shape == ((N + 15) // 16, S)
    ref = o.vote_ok.reshape(N // 16, 16, S).sum(axis=1)
    mism = np.nonzero(grp != ref)
    assert mism[0].size == 0, f"group counts differ at (group, v-1) {list(zip(*mism))[:8]}"


@pytest.mark.parametrize("name,N", [("c4", 131_072), ("c5", 65_536)])
@pytest.mark.parametrize("tie", [0, 1])
def test_vote_stage_multiwave(rk, name, N, tie):
    c, gcfg, ocfg = cfgs(rk, name)
    K, C = c["K"], c["C"]
    S, ldc = (1 << K) - 1, (C + 3) // 4 * 4
    seed = 3 + tie
    y = gen.labels(seed, 0, N, C)
    L = gen.logits(seed, 0, N, K, C, y=y)
    rank = np.random.default_rng(seed).permutation(K).astype(np.int32)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, member_rank=rank, tie=tie)
    dl = torch.empty((N, K, ldc), dtype=torch.float32, device="cuda")
    dy = torch.from_numpy(y).cuda()
    gen.dev_logits(seed, 0, N, K, C, ldc, dl.data_ptr(), dy.data_ptr())  # bit-identical to the host fill
    ctx.score_logits(dl, ldc, N, 0)
    t = ctx.subset_stats(dy, gcfg)
    o = oracle.table(L, y, K, C, tie=tie, rank=rank, cfg=ocfg, want_bits=True)
    assert t["N"] == N
    compare_tables(t, o, K=K)
    check_groups(ctx, o, N, S)


@pytest.mark.parametrize("tie", [0, 1])
def test_heads_multiwave_c4(rk, tie):
    c, gcfg, ocfg = cfgs(rk, "c4")
    K, C, D = c["K"], c["C"], c["D"]
    N = 16_384
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    y = gen.labels(9, 0, N, C)
    X = gen.features(9, 0, N, D, C, psig, False, y=y)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh, tie=tie)
    ctx.score(torch.from_numpy(X).cuda(), N)
    t = ctx.subset_stats(torch.from_numpy(y).cuda(), gcfg)
    ref = oracle.logits_gemm(X, W, b, sh)
    o = oracle.table(ref, y, K, C, tie=tie, cfg=ocfg, want_bits=True)
    compare_tables(t, o, K=K)
    check_groups(ctx, o, N, (1 << K) - 1)
    # the averaging kernel's row skipping (second-largest-logit proof) was exercised on this workload
    work, _, skipped = ctx.vote_diag()
    assert work > 0 and 0 < skipped < work * K
