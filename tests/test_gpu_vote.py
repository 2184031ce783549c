"""GPU parity of the vote stage (rk_score_logits -> rk_subset_*) against the CPU oracle.

Parity classes: P1 votes / counts / batch moments bit-exact in both tie modes;
P2 averaged-probability counts exact except oracle-flagged ambiguous pairs, avg vectors <= 1e-5
relative; P5 shard/chunk additivity bit-exact; P6 rewards <= 1e-5 relative.
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_vote(rk, L, y, K, C, tie=0, rank=None, cfg=None, offset=0):
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, member_rank=rank, tie=tie)
    dl = dev(L)
    ctx.score_logits(dl, L.shape[2], L.shape[0], offset)
    t = ctx.subset_stats(dev(y), cfg)
    torch.cuda.synchronize()
    return t, ctx


CASES = [  # (K, C, N, seed)
    (3, 10, 1000, 1),     # config c1 shape
    (3, 1000, 700, 2),    # c2 shape (K=3, C=1000), ragged N
    (6, 1000, 300, 3),    # c3 shape
    (8, 1000, 150, 4),    # c4 shape
    (12, 100, 70, 5),     # c5 shape (4095 subsets)
    (9, 50, 300, 8),      # K = 9..11: every word count of the bit-sliced vote (16..64 words)
    (10, 20, 200, 9),
    (11, 100, 150, 10),
    (12, 1000, 40, 15),   # K = 12 with C = 1000: rows do not fit twice, single-buffered CTA kernel
    (10, 1024, 50, 16),   # the widest rows of the register/shared-memory kernels
    (3, 2000, 400, 17),   # C > 1024 (SURVEY.md §8(b) allows C <= 65535): fp64 CTA averaging kernel
    (10, 1500, 80, 18),   # C > 1024 with K >= 9
    (2, 65535, 24, 19),   # the largest C of the contract
    (1, 2, 33, 6),        # degenerate: one model, two classes
    (5, 37, 517, 7),      # odd sizes, ragged everything
]


@pytest.mark.parametrize("K,C,N,seed", CASES)
@pytest.mark.parametrize("tie", [0, 1])
def test_vote_stage_parity(rk, K, C, N, seed, tie):
    y = gen.labels(seed, 0, N, C)
    L = gen.logits(seed, 0, N, K, C, y=y)
    rank = np.random.default_rng(seed).permutation(K).astype(np.int32)
    gcfg, ocfg = default_cfg(K)
    t, _ = run_vote(rk, L, y, K, C, tie=tie, rank=rank, cfg=gcfg)
    o = oracle.table(L, y, K, C, tie=tie, rank=rank, cfg=ocfg)
    assert t["N"] == N
    compare_tables(t, o, K=K)


def test_integer_logits_ties(rk):
    """Integer-valued logits: many exact top-1 ties and exact average ties (ambiguous pairs)."""
    K, C, N = 5, 6, 2000
    rng = np.random.default_rng(11)
    L = rng.integers(0, 3, size=(N, K, 8)).astype(np.float32)
    L[:, :, C:] = np.nan
    y = rng.integers(0, C, N).astype(np.int32)
    for tie in (0, 1):
        t, _ = run_vote(rk, L, y, K, C, tie=tie)
        o = oracle.table(L, y, K, C, tie=tie)
        compare_tables(t, o, K=K, check_moments=False)
        assert o.n_amb.sum() > 0  # the case is exercised


@pytest.mark.parametrize("K,C", [(4, 300), (10, 300), (4, 2000)])
def test_overflow_candidates_all_equal_rows(rk, K, C):
    """Rows with equal logits make every class a candidate (smem overflow paths; K = 10: more than 32
    competitors, the CTA kernel hands the sample to the batch kernel; C = 2000: the wide-row kernel's
    candidate list overflows and it sweeps every class)."""
    N = 64
    rng = np.random.default_rng(3)
    L = gen.logits(3, 0, N, K, C)
    L[::2, 1:, :C] = 0.0  # half the samples: models 1.. flat
    L[::4, :, :C] = rng.normal(0, 1e-3, size=(len(L[::4]), K, C)).astype(np.float32)
    y = rng.integers(0, C, N).astype(np.int32)
    t, _ = run_vote(rk, L, y, K, C)
    o = oracle.table(L, y, K, C)
    compare_tables(t, o, K=K, check_moments=False)


@pytest.mark.parametrize("cols", [4, 8])
def test_cta_average_overflow_route(rk, monkeypatch, cols):
    """K >= 9: samples whose table columns exceed the CTA averaging kernel's capacity go to the batch
    averaging kernel; a small capacity (RK_CTA_AVG_COLS, read at context creation) routes most worklist
    samples there on the c5 shape, so both kernels are held to the oracle on the same data."""
    K, C, N, seed = 12, 100, 120, 25
    monkeypatch.setenv("RK_CTA_AVG_COLS", str(cols))
    y = gen.labels(seed, 0, N, C)
    L = gen.logits(seed, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)


@pytest.mark.parametrize("cap", [1, 5])
def test_pair_list_full(rk, monkeypatch, cap):
    """K >= 9, C <= 128: near-tie (sample, subset) pairs go to the fp64 pair kernel; when the list is full
    the warp kernel hands the whole sample to the CTA kernel and marks its reserved slots as skipped
    (RK_PAIR_CAP shrinks the list). Ties are forced with integer logits."""
    K, C, N = 10, 8, 300
    monkeypatch.setenv("RK_PAIR_CAP", str(cap))
    rng = np.random.default_rng(27)
    L = rng.integers(0, 3, size=(N, K, C)).astype(np.float32)
    y = rng.integers(0, C, N).astype(np.int32)
    gcfg, ocfg = default_cfg(K)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)
    assert t["n_recheck"].sum() > 0


@pytest.mark.parametrize("K", [8, 12])
def test_tiny_label_probabilities(rk, K):
    """Steep logits (x40 on every third sample): p[m][y] underflows fp32 for some models, so subset sums
    of y can be (nearly) subnormal; those decisions must still match the fp64 oracle."""
    C, N, seed = 100, 90, 26
    y = gen.labels(seed, 0, N, C)
    L = gen.logits(seed, 0, N, K, C, y=y)
    L[::3] *= 40.0
    gcfg, ocfg = default_cfg(K)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)


@pytest.mark.parametrize("K", [4, 11])
def test_chunked_and_sharded_equal_one_shot(rk, K):
    """Streaming chunks (multiples of lcm(B)) and disjoint shards sum to the one-shot table (I7, P5)."""
    C, N = 100, 1000
    y = gen.labels(21, 0, N, C)
    L = gen.logits(21, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K, B=(16, 32, 64))
    o = oracle.table(L, y, K, C, cfg=ocfg)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C)
    ctx.subset_reset(gcfg)
    keep = []  # the library borrows the logits pointer until the next rk_score*: keep buffers alive
    for off, n in [(0, 256), (256, 512), (768, 232)]:
        keep.append(dev(L[off:off + n]))
        ctx.score_logits(keep[-1], L.shape[2], n, off)
        ctx.subset_accumulate(dev(y[off:off + n]))
    t = ctx.subset_finalize()
    compare_tables(t, o, K=K)
    # two independent "ranks" (world=1 contexts) on disjoint shards: integer tables add exactly
    parts = []
    for off, n in [(0, 512), (512, 488)]:
        c2 = rk.Context(0)
        c2.load_ensemble(K, C)
        keep.append(dev(L[off:off + n]))
        c2.score_logits(keep[-1], L.shape[2], n, off)
        parts.append(c2.subset_stats(dev(y[off:off + n]), gcfg))
    for k in ("cnt_vote", "corr", "O", "Q", "E"):
        np.testing.assert_array_equal(parts[0][k] + parts[1][k], getattr(o, k), err_msg=k)


@pytest.mark.parametrize("B,N", [((16, 48, 80), 1000),   # non-nested sizes, L = 240, staged overdue table
                                 ((1, 4096), 9000),       # gs = 1, L = 4096: per-chunk table > 32 KB, global path
                                 ((3, 6, 12), 61)])       # ragged tail, gs = 1
@pytest.mark.parametrize("K", [4, 10])  # K = 10: warp-per-chunk vote kernel, vote totals summed by the q pass
def test_labelled_moments_batch_sets(rk, B, N, K):
    C = 50
    y = gen.labels(31, 0, N, C)
    L = gen.logits(31, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K, B=B, tau_ns=100_000_000)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)
    assert o.Q.sum() > 0  # the labelled moments are exercised


@pytest.mark.parametrize("K,rates", [(5, (64.0, 128.0, 572.0, 1144.0)),
                                     (9, (40.0, 64.0, 128.0, 300.0, 572.0, 1144.0))])  # 6 rates: 8-wide vectors
def test_labelled_moments_doubling_batches(rk, K, rates):
    """The bench's doubling batch sizes {16, ..., 256} take the pairwise-sum tree kernel for Q; ragged N."""
    C, N = 40, 2000
    B = (16, 32, 64, 128, 256)
    y = gen.labels(41, 0, N, C)
    L = gen.logits(41, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K, B=B, rates=rates)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)


def test_arrival_ns_input(rk):
    K, C, N = 3, 10, 640
    y = gen.labels(5, 0, N, C)
    L = gen.logits(5, 0, N, K, C, y=y)
    arr = np.cumsum(np.random.default_rng(0).integers(0, 40_000_000, N)).astype(np.int64)
    import paper_1804_06087_b200 as m
    gcfg, ocfg = default_cfg(K)
    gcfg = m.RewardCfg(B=gcfg.B, beta=0.5, tau_ns=300_000_000, lat_ns=gcfg.lat_ns, arrival_ns=arr)
    ocfg = oracle.RewardCfg(B=ocfg.B, beta=0.5, tau_ns=300_000_000, lat_ns=ocfg.lat_ns, arrival_ns=arr)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)


def test_predict_parity(rk):
    K, C, N = 4, 50, 300
    y = gen.labels(8, 0, N, C)
    L = gen.logits(8, 0, N, K, C, y=y)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, tie=0)
    dl = dev(L)
    ctx.score_logits(dl, L.shape[2], N)
    for v in (1, 5, 15):
        pv = torch.empty(N, dtype=torch.int32, device="cuda")
        pa = torch.empty(N, dtype=torch.int32, device="cuda")
        ap = torch.empty((N, C), dtype=torch.float32, device="cuda")
        ctx.predict(v, pv, pa, ap)
        opv, opa, oap, _, _ = oracle.predict(L, K, C, v, want_avgprob=True)
        np.testing.assert_array_equal(pv.cpu().numpy(), opv)
        np.testing.assert_allclose(ap.cpu().numpy(), oap, rtol=1e-5, atol=1e-7)  # I4 at 1e-5
        srt = np.sort(oap, axis=1)
        clear = (srt[:, -1] - srt[:, -2]) > 1e-5 * srt[:, -1]
        np.testing.assert_array_equal(pa.cpu().numpy()[clear], opa[clear])
    with pytest.raises(rk.RkError):
        ctx.predict(0)


def test_errors(rk):
    K, C, N = 3, 10, 64
    y = gen.labels(1, 0, N, C)
    L = gen.logits(1, 0, N, K, C, y=y)
    bad = L.copy()
    bad[5, 1, 3] = np.nan
    with pytest.raises(rk.RkError) as e:
        run_vote(rk, bad, y, K, C)
    assert e.value.status == 7  # RK_ENONFINITE
    yy = y.copy()
    yy[3] = C
    with pytest.raises(rk.RkError) as e:
        run_vote(rk, L, yy, K, C)
    assert e.value.status == 6  # RK_ELABEL
    ok = L.copy()
    ok[5, 1, 3] = -np.inf  # legal
    run_vote(rk, ok, y, K, C)
    # empty batch
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C)
    with pytest.raises(rk.RkError) as e:  # nothing scored yet
        ctx.outputs_s2()
    assert e.value.status == 2  # RK_ESTATE
    ctx.score_logits(None, 12, 0)
    assert ctx.outputs_s2() is None  # caller logits: no second-largest logits, no row skipping
    t = ctx.subset_stats(None)
    assert t["N"] == 0 and t["cnt_vote"].sum() == 0
    assert ctx.vote_diag() == (0, 0, 0)


QUEUE_CASES = [(3, 10, 1000, 11), (8, 1000, 300, 12), (12, 100, 200, 13), (5, 37, 517, 14)]


@pytest.mark.parametrize("K,C,N,seed", QUEUE_CASES)
def test_queue_mode_parity(rk, K, C, N, seed):
    """Reading Q15: FIFO finish times; the rates span under- and overload."""
    y = gen.labels(seed, 0, N, C)
    L = gen.logits(seed, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K, rates=(64.0, 572.0, 4000.0), queue=True)
    t, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    compare_tables(t, o, K=K)
    _, onq = default_cfg(K, rates=(64.0, 572.0, 4000.0))
    o0 = oracle.table(L, y, K, C, cfg=onq)
    assert (o.O > o0.O).any()  # the backlog matters in this workload


def test_queue_mode_chunks_and_shards(rk):
    """Backlog carried across in-order chunks; a shard starting at sample 512 derives the backlog of
    the earlier batches from the rates; shards add up to the one-shot table."""
    K, C, N = 4, 100, 1000
    y = gen.labels(22, 0, N, C)
    L = gen.logits(22, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K, B=(16, 32, 64), rates=(300.0, 2000.0), queue=True)
    o = oracle.table(L, y, K, C, cfg=ocfg)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C)
    ctx.subset_reset(gcfg)
    keep = []
    for off, n in [(0, 256), (256, 512), (768, 232)]:
        keep.append(dev(L[off:off + n]))
        ctx.score_logits(keep[-1], L.shape[2], n, off)
        ctx.subset_accumulate(dev(y[off:off + n]))
    compare_tables(ctx.subset_finalize(), o, K=K)
    parts = []
    for off, n in [(0, 512), (512, 488)]:
        c2 = rk.Context(0)
        c2.load_ensemble(K, C)
        keep.append(dev(L[off:off + n]))
        c2.score_logits(keep[-1], L.shape[2], n, off)
        parts.append(c2.subset_stats(dev(y[off:off + n]), gcfg))
    for k in ("O", "Q", "E"):
        np.testing.assert_array_equal(parts[0][k] + parts[1][k], getattr(o, k), err_msg=k)
    # out-of-order chunks are rejected; caller arrivals need the stream to start at sample 0
    ctx.subset_reset(gcfg)
    ctx.score_logits(keep[1], L.shape[2], 512, 256)
    ctx.subset_accumulate(dev(y[256:768]))
    ctx.score_logits(keep[0], L.shape[2], 256, 0)
    with pytest.raises(rk.RkError):
        ctx.subset_accumulate(dev(y[:256]))
    import paper_1804_06087_b200 as m
    arr = np.arange(N, dtype=np.int64) * 1_000_000
    acfg = m.RewardCfg(B=[16], beta=1.0, tau_ns=10_000_000, lat_ns=gcfg.lat_ns[:, :1].copy(), arrival_ns=arr[512:],
                       queue=True)
    c3 = rk.Context(0)
    c3.load_ensemble(K, C)
    c3.score_logits(keep[-1], L.shape[2], 488, 512)
    with pytest.raises(rk.RkError) as e:
        c3.subset_stats(dev(y[512:]), acfg)
    assert e.value.status == 8  # RK_EUNSUPPORTED


def test_nccl_path_single_rank(rk):
    """A6 over NCCL with a one-rank communicator: the all-reduce code path runs (profiled launch) and
    the table equals the communicator-free one (this environment exposes one GPU per call)."""
    K, C, N = 5, 100, 768
    y = gen.labels(41, 0, N, C)
    L = gen.logits(41, 0, N, K, C, y=y)
    gcfg, ocfg = default_cfg(K)
    t0, _ = run_vote(rk, L, y, K, C, cfg=gcfg)
    c = rk.Context(0, 0, 1, rk.nccl_unique_id())
    c.load_ensemble(K, C)
    dl = dev(L)
    c.score_logits(dl, L.shape[2], N)
    c.set_profiling(True)
    t1 = c.subset_stats(dev(y), gcfg)
    assert c.kernel_stats()["nccl_allreduce"]["launches"] == 1
    for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E", "reward_sur", "reward_lab"):
        np.testing.assert_array_equal(t1[k], t0[k], err_msg=k)
    compare_tables(t1, oracle.table(L, y, K, C, cfg=ocfg), K=K)
