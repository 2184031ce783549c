"""GPU parity of the tcgen05 head GEMM (rk_score, A1+A2) and of the end-to-end path.

P3: integer-exact mode (X, W in {-1,0,1}, integer bias, scale 2^-k): logits bit-exact, hence votes
and counts bit-exact end to end. P4: real-valued bf16 mode: |dlogit| <= c * D * 2^-24 * sum|x*w|.
"""
import numpy as np
import pytest

import gen
import oracle
from gpu_helpers import compare_tables, default_cfg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def make(K, C, D, N, seed, real, bias=True):
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = gen.labels(seed, 0, N, C)
    X = gen.features(seed, 0, N, D, C, psig, real, y=y)
    W = gen.weights(seed + 100, K, C, D, f0, df, real)
    b = gen.bias(seed + 200, K, C, real) if bias else None
    return y, X, W, b, sh


def run_gemm(rk, K, C, D, N, X, W, b, sh, tie=0):
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), None if b is None else torch.from_numpy(b).cuda(), sh,
                      tie=tie)
    ctx.score(torch.from_numpy(X).cuda(), N)
    out = ctx.outputs()
    ldc = out["ldc"]
    torch.cuda.synchronize()
    lg = dev_view(out["logits"], (N, K, ldc), "<f4")
    t1 = dev_view(out["top1"], (N, K), "<i4")
    mx = dev_view(out["rmax"], (N, K), "<f4")
    ls = dev_view(out["lsum"], (N, K), "<f4")
    return ctx, lg, t1, (mx, ls)


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3}


def dev_view(ptr, shape, typestr):
    """Copy a library-owned device buffer to a host numpy array."""
    return torch.as_tensor(_CAI(ptr, shape, typestr), device="cuda").cpu().numpy()


@pytest.mark.parametrize("K,C,D,N", [(3, 10, 128, 200), (2, 100, 256, 300), (3, 1000, 512, 130),
                                     (12, 100, 1024, 257), (1, 2, 64, 5), (4, 300, 192, 129), (2, 2000, 256, 300)])
@pytest.mark.parametrize("cluster", ["1", "2"])
def test_int_mode_bit_exact(rk, K, C, D, N, cluster, monkeypatch):
    monkeypatch.setenv("RK_GEMM_CLUSTER", cluster)  # read by rk_create: 1 CTA or 2-CTA W multicast
    y, X, W, b, sh = make(K, C, D, N, 3, real=False)
    ctx, lg, t1, ls = run_gemm(rk, K, C, D, N, X, W, b, sh)
    ref = oracle.logits_gemm(X, W, b, sh)  # fp64, exact for these integer inputs
    np.testing.assert_array_equal(lg[:, :, :C], ref.astype(np.float32))
    np.testing.assert_array_equal(t1, np.argmax(ref, axis=2))
    check_row_stats(ls, ref)
    # second-largest logit (the averaging kernel's row-skip proof): per-model epilogue only (Cp > 128);
    # ties at the maximum are frequent on this integer grid, where it must equal the maximum
    p2 = ctx.outputs_s2()
    if (C + 15) // 16 * 16 > 128:
        s2 = dev_view(p2, (N, K), "<f4")
        np.testing.assert_array_equal(s2, np.sort(ref, axis=2)[:, :, -2].astype(np.float32))
    else:
        assert p2 is None


def check_row_stats(stats, ref):
    """rmax bit-exact (fp32 of the exact logits); lsum = log sum_c exp(l - max) = oracle lse - max within
    4e-6 absolute (fp32 sum of ex2.approx terms; relative to the max, so the bound does not grow with the
    logits' offset -- the p[m][c] the averaging kernels form from it are within ~4e-6 relative, inside
    the 2e-5 fp64-recheck band). The error of a recursive fp32 sum grows with its number of
    terms (Higham: (n-1)u worst case), so rows wider than 1000 classes get a proportionally wider bound;
    those rows (ldc > 1024) are averaged by the fp64 wide-row kernel, which recomputes the normaliser, and
    lsum only feeds the theta pruning there, whose threshold keeps a 1e-3 log margin (rk_internal.h)."""
    mx, ls = stats
    N, K = mx.shape
    C = ref.shape[2]
    np.testing.assert_array_equal(mx, ref.max(axis=2).astype(np.float32))
    ref_ls = np.array([[oracle.lse(ref[n, m]) - ref[n, m].max() for m in range(K)] for n in range(N)])
    np.testing.assert_allclose(ls, ref_ls, rtol=0, atol=4e-6 * max(1.0, C / 1000))


def test_real_mode_tolerance(rk):
    K, C, D, N = 3, 1000, 1024, 300
    y, X, W, b, sh = make(K, C, D, N, 5, real=True)
    ctx, lg, t1, ls = run_gemm(rk, K, C, D, N, X, W, b, sh)
    ref = oracle.logits_gemm(X, W, b, sh)
    absum = np.einsum("nd,kcd->nkc", np.abs(gen.bf16_to_f64(X)), np.abs(gen.bf16_to_f64(W))) * 2.0**sh
    bound = 4 * D * 2.0**-24 * absum + 2.0**-24 * np.abs(ref)
    err = np.abs(lg[:, :, :C].astype(np.float64) - ref)
    assert (err <= bound).all(), float((err / np.maximum(bound, 1e-30)).max())
    # top-1 exact except where the oracle's top-2 logit gap is within the bound (flagged)
    srt = np.sort(ref, axis=2)
    gap = srt[:, :, -1] - srt[:, :, -2]
    clear = gap > 2 * bound.max(axis=2)
    np.testing.assert_array_equal(t1[clear], np.argmax(ref, axis=2)[clear])


@pytest.mark.parametrize("K,C,D,N,tie", [(3, 1000, 512, 600, 0), (8, 1000, 256, 150, 1), (12, 100, 512, 64, 0),
                                         (3, 2000, 256, 300, 1)])
def test_end_to_end_int_mode(rk, K, C, D, N, tie):
    """X -> tcgen05 heads -> vote/average/moments -> reward table equals the oracle on its own fp64 logits."""
    y, X, W, b, sh = make(K, C, D, N, 9, real=False)
    ctx = rk.Context(0)
    rank = np.random.default_rng(1).permutation(K).astype(np.int32)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh, member_rank=rank, tie=tie)
    gcfg, ocfg = default_cfg(K)
    ctx.score(torch.from_numpy(X).cuda(), N)
    t = ctx.subset_stats(torch.from_numpy(y).cuda(), gcfg)
    ref = oracle.logits_gemm(X, W, b, sh)
    o = oracle.table(ref, y, K, C, tie=tie, rank=rank, cfg=ocfg)
    compare_tables(t, o, K=K)


def test_host_buffers_e2e(rk):
    """Host (numpy) X and labels are staged by the library (the e2e path bench.py times)."""
    K, C, D, N = 3, 100, 256, 500
    y, X, W, b, sh = make(K, C, D, N, 13, real=False)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, W, b, sh)
    ctx.score(X, N)
    t = ctx.subset_stats(y, None)
    o = oracle.table(oracle.logits_gemm(X, W, b, sh), y, K, C)
    compare_tables(t, o, K=K, check_moments=False)


def test_host_buffers_chunked(rk):
    """Host X large enough for the library's chunked staging (copies overlapping the GEMM chunks, the
    trailing chunk split into quarter pieces): the table equals the device-X table of the same inputs."""
    K, C, D, N = 3, 300, 128, 150_000
    y, X, W, b, sh = make(K, C, D, N, 14, real=False)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, W, b, sh)
    ctx.score(torch.from_numpy(X).cuda(), N)
    t_dev = ctx.subset_stats(torch.from_numpy(y).cuda(), None)
    ctx.score(X, N)  # host numpy X: staged by the library in chunks
    t_host = ctx.subset_stats(y, None)
    for k in ("cnt_vote", "cnt_avg", "n_recheck"):
        np.testing.assert_array_equal(t_host[k], t_dev[k], err_msg=k)
    assert t_host["N"] == N
