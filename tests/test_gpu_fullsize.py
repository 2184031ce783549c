"""Full-size parity at BASELINE.json's sizes, in bench.py's launch configuration.

c4 (K=8, C=1000, N=1,000,000, D=2048) and c5 (K=12, C=100, N=4,000,000, D=1024) run through the
calls bench.py times: rk_score on device-generated X (integer mode), then rk_subset_stats with the
bench's reward configuration, one launch over all N. The oracle cannot process 10^6 samples in a
test, so parity at this size is checked on sampled outputs and through properties that hold at any
size:

  1. heads (A1/A2) on sampled rows: the oracle recomputes the logits in fp64 from the same seeded
     inputs (exact in integer mode) -> logits, top-1 and row max bit-exact, lsum within 2e-6;
  2. per-sample subset decisions (A3/A4) on the sampled rows via rk_predict(v) at full size, against
     oracle.predict on the oracle's own logits (votes exact; averages exact where the top-2 gap of the
     oracle's average exceeds 1e-5 relative);
  3. invariant I1 at full size: for a single-model subset {m}, vote and average counts both equal the
     number of samples whose top-1 of model m is the label;
  4. additivity (P5) at full size: the one-launch table equals the sum of the tables of four
     lcm(B)-aligned shards scored by separate contexts, bit-exact for every integer section (a
     self-consistency check; the oracle comparison of whole tables at multi-wave sizes of these
     shapes -- c4 N = 131,072, c5 N = 65,536 -- is tests/test_gpu_multiwave.py);
  5. fold (A7) of the full-size table: rewards equal eq. `multi_acc_reward` applied
     to the returned integer sections;
  6. c4: the averaging kernel's row skipping (rows the GEMM's second-largest logit proves irrelevant are
     not streamed) leaves the full-size table unchanged: the same logits through rk_score_logits, where
     every row is streamed, give the identical table;
  7. c4: the NEXT-3 fused path (rk_score_labelled) at full size gives the identical table as well.
"""
import numpy as np
import pytest

import gen
import oracle
from bench import BETA, CONFIGS, TAU_NS, lat_profile
from test_gpu_gemm import check_row_stats

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3}


def dev_rows(ptr, row_shape, typestr, itemsize, rows):
    """Copy selected rows of a library-owned [N][...] device buffer to host."""
    n_per = int(np.prod(row_shape))
    out = []
    for r0, r1 in rows:
        t = torch.as_tensor(_CAI(ptr + r0 * n_per * itemsize, (r1 - r0,) + tuple(row_shape), typestr), device="cuda")
        out.append(t.cpu().numpy())
    return np.concatenate(out)


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def bench_setup(rk, name):
    c = CONFIGS[name]
    K, C, D, N = c["K"], c["C"], c["D"], c["N"]
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    labels = torch.empty(N, dtype=torch.int32, device="cuda")
    X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
    gen.dev_labels(1, 0, N, C, labels.data_ptr())
    gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), labels.data_ptr())
    cfg = rk.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat_profile(K, c["B"]), rates=c["rates"],
                       want_exceed=True, want_labelled=True)
    return c, (W, b, sh, psig), X, labels, cfg


def sampled_blocks(N, nblk=2, blk=64, seed=7):
    rng = np.random.default_rng(seed)
    starts = sorted(rng.choice(N // blk, size=nblk, replace=False) * blk)
    return [(int(s), int(s) + blk) for s in starts]


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_fullsize(rk, name):
    c, (W, b, sh, psig), X, labels, cfg = bench_setup(rk, name)
    K, C, D, N = c["K"], c["C"], c["D"], c["N"]
    S = (1 << K) - 1
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, W, b, sh)
    ctx.score(X, N)
    t = ctx.subset_stats(labels, cfg)
    torch.cuda.synchronize()
    assert t["N"] == N

    # 1. sampled heads
    blocks = sampled_blocks(N)
    out = ctx.outputs()
    ldc = out["ldc"]
    lg = dev_rows(out["logits"], (K, ldc), "<f4", 4, blocks)
    t1 = dev_rows(out["top1"], (K,), "<i4", 4, blocks)
    mx = dev_rows(out["rmax"], (K,), "<f4", 4, blocks)
    ls = dev_rows(out["lsum"], (K,), "<f4", 4, blocks)
    y = np.concatenate([gen.labels(1, r0, r1 - r0, C) for r0, r1 in blocks])
    Xs = np.concatenate([gen.features(1, r0, r1 - r0, D, C, psig, False, y=gen.labels(1, r0, r1 - r0, C))
                         for r0, r1 in blocks])
    ref = oracle.logits_gemm(Xs, W, b, sh)
    np.testing.assert_array_equal(lg[:, :, :C], ref.astype(np.float32))
    np.testing.assert_array_equal(t1, np.argmax(ref, axis=2))
    check_row_stats((mx, ls), ref)

    # 2. per-sample decisions at full size for several subsets
    for v in sorted({1, 3, (1 << K) - 1, 0b101101 & S, S ^ 1}):
        pv = torch.empty(N, dtype=torch.int32, device="cuda")
        pa = torch.empty(N, dtype=torch.int32, device="cuda")
        ctx.predict(v, pv, pa)
        idx = np.concatenate([np.arange(r0, r1) for r0, r1 in blocks])
        gpv, gpa = pv.cpu().numpy()[idx], pa.cpu().numpy()[idx]
        opv, opa, oap, _, _ = oracle.predict(ref.astype(np.float32), K, C, v, want_avgprob=True)
        np.testing.assert_array_equal(gpv, opv, err_msg=f"vote v={v}")
        srt = np.sort(oap, axis=1)
        clear = (srt[:, -1] - srt[:, -2]) > 1e-5 * srt[:, -1]
        np.testing.assert_array_equal(gpa[clear], opa[clear], err_msg=f"avg v={v}")

    # 3. I1 at full size
    top_all = torch.as_tensor(_CAI(out["top1"], (N, K), "<i4"), device="cuda")
    for m in range(K):
        n_ok = int((top_all[:, m] == labels).sum().item())
        assert t["cnt_vote"][(1 << m) - 1] == n_ok
        assert t["cnt_avg"][(1 << m) - 1] == n_ok

    # 4. additivity over four aligned shards (separate contexts, same launch configuration per shard)
    from paper_1804_06087_b200.shard import shard_ranges
    acc = None
    for off, n in shard_ranges(N, 4, c["B"]):
        c2 = rk.Context(0)
        c2.load_ensemble(K, C, D, W, b, sh)
        c2.score(X[off:off + n], n, off)
        part = c2.subset_stats(labels[off:off + n], cfg)
        torch.cuda.synchronize()
        acc = part if acc is None else {k: acc[k] + part[k] for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E")}
        c2.close()
    for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E"):
        np.testing.assert_array_equal(acc[k], t[k], err_msg=k)

    # 6. (K <= 8) the averaging kernel's row skipping and worklist records at full size: the same logits fed
    #    back through rk_score_logits (statistics recomputed by the classify kernel, no second-largest
    #    logit -> every row streamed) give the same table
    if K <= 8:
        work, _, skipped = ctx.vote_diag()
        assert 0 < skipped < work * K
        ctx.score_logits(torch.as_tensor(_CAI(out["logits"], (N, K, ldc), "<f4"), device="cuda"), ldc, N, 0)
        t2 = ctx.subset_stats(labels, cfg)
        torch.cuda.synchronize()
        assert ctx.vote_diag()[2] == 0
        for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E"):
            np.testing.assert_array_equal(t2[k], t[k], err_msg=f"row skipping changed {k}")

    # 7. (K <= 8) NEXT-3 at full size: the fused forward + vote (rk_score_labelled: top-16 lists with the
    #    carried thresholds of every thread across its many work units, sparse averages, recompute fallback)
    #    gives the same table as the logits path
    if K <= 8:
        cf = rk.Context(0)
        cf.load_ensemble(K, C, D, W, b, sh)
        cf.score_labelled(X, labels, N)
        tf = cf.subset_stats(labels, cfg)
        torch.cuda.synchronize()
        for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E"):
            np.testing.assert_array_equal(tf[k], t[k], err_msg=f"fused path changed {k}")
        work, fb, _ = cf.vote_diag()
        assert 0 < fb < work
        cf.close()

    # 5. fold of the full-size integer table (eq. multi_acc_reward; readings Q7, Q11, Q13)
    B = np.array(c["B"], dtype=np.float64)
    nb = np.array([N // bb for bb in c["B"]], dtype=np.float64)
    a = t["cnt_vote"].astype(np.float64) / N
    sur = a[None, None, :] * (nb[None, :, None] * B[None, :, None] - BETA * t["O"].astype(np.float64))
    lab = t["corr"].astype(np.float64)[None, :, :] - (BETA / B)[None, :, None] * t["Q"].astype(np.float64)
    np.testing.assert_allclose(t["reward_sur"], sur, rtol=1e-12)
    np.testing.assert_allclose(t["reward_lab"], lab, rtol=1e-12, atol=1e-9)
    ctx.close()
