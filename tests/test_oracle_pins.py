"""Pins for the CPU oracle (oracle/) against things other than itself.

* golden hand-computed examples (tests/golden/, each with its citation): W1-W4, R1-R5;
* closed forms (rational softmax, exact Fraction averages);
* library routines (numpy argmax/bincount first-occurrence semantics, torch.softmax);
* an independently written brute-force formulation of the vote (member-pair support
  counting, not the oracle's class histogram) over every prediction tuple for tiny K, C;
* invariants I1-I8.
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read(name):
    rows = []
    for ln in open(os.path.join(GOLD, name)):
        ln = ln.strip()
        if ln and not ln.startswith("#"):
            rows.append(ln.split())
    return rows


def onehot_logits(preds, C):
    """fp32 logits whose top-1 is exactly `preds` (one row per model)."""
    N, K = preds.shape
    L = np.zeros((N, K, C), np.float32)
    for n in range(N):
        for m in range(K):
            L[n, m, preds[n, m]] = 1.0
    return L


# ---------------------------------------------------------------- W1 (vote tie rules)
def _w1():
    rows = _read("w1_vote_tiebreak.txt")
    K = int(rows[0][1]); C = int(rows[1][1])
    data = [r for r in rows[2:] if r[0].lstrip("-").isdigit()]
    arr = np.array(data, dtype=np.int32)
    preds, y = arr[:, :K], arr[:, K]
    exp = {r[0]: np.array(r[1:], dtype=np.uint64) for r in rows if not r[0].lstrip("-").isdigit() and r[0] not in "KC"}
    return K, C, preds, y, exp


def test_w1_counts_both_tie_modes():
    K, C, preds, y, exp = _w1()
    L = onehot_logits(preds, C)
    tb = oracle.table(L, y, K, C, tie=oracle.TIE_BEST_MEMBER)
    tl = oracle.table(L, y, K, C, tie=oracle.TIE_LOWEST_CLASS)
    assert tb.cnt_vote.tolist() == exp["best_member"].tolist()
    assert tl.cnt_vote.tolist() == exp["lowest_class"].tolist()


def test_w1_per_sample_bits_mask3():
    K, C, preds, y, exp = _w1()
    for tie, key in ((oracle.TIE_BEST_MEMBER, "mask3_best_member"), (oracle.TIE_LOWEST_CLASS, "mask3_lowest_class")):
        bits = [int(oracle.vote(preds[n], 3, C, tie) == y[n]) for n in range(len(y))]
        assert bits == exp[key].astype(int).tolist()


def test_w1_table_bits_mask3():
    """The table's per-sample vote bits (want_bits, used for the per-group parity of the GPU's group
    counts) reproduce the hand-computed mask-3 bits, and every column sums to its cnt_vote."""
    K, C, preds, y, exp = _w1()
    L = onehot_logits(preds, C)
    for tie, key in ((oracle.TIE_BEST_MEMBER, "mask3_best_member"), (oracle.TIE_LOWEST_CLASS, "mask3_lowest_class")):
        t = oracle.table(L, y, K, C, tie=tie, want_bits=True)
        assert t.vote_ok[:, 3 - 1].astype(int).tolist() == exp[key].astype(int).tolist()
        assert t.vote_ok.sum(0).tolist() == t.cnt_vote.tolist()
        assert t.avg_ok.sum(0).tolist() == t.cnt_avg.tolist()


# ---------------------------------------------------------------- W2 (reading Q2)
def test_w2_tied_voters_reading():
    # (7,3,3,5,5): tied-voters reading -> 3; best-overall would give 7 (not a majority class).
    assert oracle.vote([7, 3, 3, 5, 5], 31, 8, oracle.TIE_BEST_MEMBER) == 3
    assert oracle.vote([7, 3, 3, 5, 5], 31, 8, oracle.TIE_LOWEST_CLASS) == 3
    # discriminates BEST_MEMBER from LOWEST_CLASS: tied classes 5 (voters m1,m2) and 3 (m3,m4)
    assert oracle.vote([7, 5, 5, 3, 3], 31, 8, oracle.TIE_BEST_MEMBER) == 5
    assert oracle.vote([7, 5, 5, 3, 3], 31, 8, oracle.TIE_LOWEST_CLASS) == 3
    # explicit ranks: make m3 the best model -> 3 wins the 2-2 tie
    assert oracle.vote([7, 5, 5, 3, 3], 31, 8, oracle.TIE_BEST_MEMBER, rank=[1, 2, 3, 0, 4]) == 3


# ---------------------------------------------------------------- W3 / W4 (softmax average)
def _fr(tok):
    a, b = tok.split("/")
    return Fraction(int(a), int(b))


def test_w3_w4_rational_softmax_and_average():
    g = {r[0]: [_fr(t) for t in r[1:]] for r in _read("w3_w4_softmax_avg.txt")}
    lA, lB, lC = np.log([1.0, 2.0, 1.0]), np.log([3.0, 1.0, 1.0]), np.log([1.0, 1.0, 3.0])
    pA, pB, pC = oracle.softmax(lA), oracle.softmax(lB), oracle.softmax(lC)
    for p, key in ((pA, "pA"), (pB, "pB"), (pC, "pC")):
        np.testing.assert_allclose(p, [float(f) for f in g[key]], rtol=1e-15, atol=1e-16)
    pred, amb, avg = oracle.avg(np.stack([pA, pB]), 3)
    np.testing.assert_allclose(avg, [float(f) for f in g["avgAB"]], rtol=1e-15)
    assert pred == 0 and not amb
    # vote {A,B}: A (model 0) predicts 1, B predicts 0 -> 1-1 tie
    tA, tB = oracle.top1(lA), oracle.top1(lB)
    assert (tA, tB) == (1, 0)
    assert oracle.vote([tA, tB], 3, 3, oracle.TIE_BEST_MEMBER) == 1
    assert oracle.vote([tA, tB], 3, 3, oracle.TIE_LOWEST_CLASS) == 0
    pred, amb, avg = oracle.avg(np.stack([pA, pB, pC]), 7)
    np.testing.assert_allclose(avg, [float(f) for f in g["avgABC"]], rtol=1e-15)
    assert amb, "exact tie 7/20 == 7/20 must be flagged ambiguous"


# ---------------------------------------------------------------- library pins
def test_top1_first_occurrence_matches_numpy():
    rng = np.random.default_rng(0)
    for _ in range(200):
        row = rng.integers(0, 4, size=rng.integers(2, 40)).astype(np.float32)  # many exact ties
        assert oracle.top1(row) == int(np.argmax(row))
        assert oracle.top1(row.astype(np.float64)) == int(np.argmax(row))


def test_softmax_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    for C in (2, 10, 1000):
        l = rng.normal(0, 4, C)
        ref = torch.softmax(torch.tensor(l, dtype=torch.float64), -1).numpy()
        np.testing.assert_allclose(oracle.softmax(l), ref, rtol=1e-13, atol=1e-300)
        ref_lse = float(torch.logsumexp(torch.tensor(l, dtype=torch.float64), -1))
        assert abs(oracle.lse(l) - ref_lse) <= 1e-13 * max(1.0, abs(ref_lse))


def test_lowest_class_vote_is_argmax_bincount():  # invariant I5
    rng = np.random.default_rng(2)
    for _ in range(500):
        K = int(rng.integers(1, 9)); C = int(rng.integers(2, 7))
        t = rng.integers(0, C, K).astype(np.int32)
        v = int(rng.integers(1, 1 << K))
        members = [t[i] for i in range(K) if (v >> i) & 1]
        assert oracle.vote(t, v, C, oracle.TIE_LOWEST_CLASS) == int(np.argmax(np.bincount(members, minlength=C)))


# ---------------------------------------------------------------- brute force, independent formulation
def _vote_pairwise(preds, v, tie, rank):
    """Member-pair support counting (no class histogram): support(i) = #{j in v: pred_j == pred_i}."""
    mem = [i for i in range(len(preds)) if (v >> i) & 1]
    sup = {i: sum(1 for j in mem if preds[j] == preds[i]) for i in mem}
    top = max(sup.values())
    tied = [i for i in mem if sup[i] == top]
    if tie == oracle.TIE_BEST_MEMBER:
        return preds[min(tied, key=lambda i: rank[i])]
    return min(preds[i] for i in tied)


@pytest.mark.parametrize("K,C", [(1, 3), (2, 4), (3, 5), (4, 4)])
def test_vote_brute_force_all_tuples(K, C):
    rng = np.random.default_rng(K * 10 + C)
    ranks = [list(range(K)), list(rng.permutation(K))]
    for preds in itertools.product(range(C), repeat=K):
        for v in range(1, 1 << K):
            for rank in ranks:
                for tie in (oracle.TIE_BEST_MEMBER, oracle.TIE_LOWEST_CLASS):
                    got = oracle.vote(list(preds), v, C, tie, rank=rank)
                    assert got == _vote_pairwise(preds, v, tie, rank), (preds, v, tie, rank)


def test_avg_exact_fraction_brute_force():
    """Dyadic probabilities -> exact Fraction average; oracle pred must equal the exact argmax
    (smallest index on exact ties) and flag exactly the near/exact ties."""
    rng = np.random.default_rng(3)
    for _ in range(400):
        K = int(rng.integers(1, 5)); C = int(rng.integers(2, 6))
        num = rng.integers(0, 9, size=(K, C)).astype(np.float64)  # frequent exact ties
        num[:, 0] += 1
        p = num / 64.0
        v = int(rng.integers(1, 1 << K))
        mem = [i for i in range(K) if (v >> i) & 1]
        exact = [sum(Fraction(int(num[i, c]), 64) for i in mem) / len(mem) for c in range(C)]
        best = max(exact)
        want = exact.index(best)
        srt = sorted(exact, reverse=True)
        pred, amb, avg = oracle.avg(p, v)
        assert amb == (srt[0] == srt[1]), (num, v)
        if not amb:
            assert pred == want
        np.testing.assert_allclose(avg, [float(e) for e in exact], rtol=1e-15)


# ---------------------------------------------------------------- invariants on generated data
def _data(K, C, N, seed=1):
    y = gen.labels(seed, 0, N, C)
    L = gen.logits(seed, 0, N, K, C, y=y)
    return L, y


@pytest.mark.parametrize("K,C", [(3, 10), (4, 100), (5, 30)])
def test_I1_singletons_equal_model_accuracy(K, C):
    L, y = _data(K, C, 600)
    t = oracle.table(L, y, K, C)
    for m in range(K):
        acc = int((np.argmax(L[:, m, :C], axis=1) == y).sum())
        assert t.cnt_vote[(1 << m) - 1] == acc
        assert t.cnt_avg[(1 << m) - 1] == acc


def test_I2_pairs():
    K, C = 4, 10
    L, y = _data(K, C, 800, seed=4)
    top = np.argmax(L[:, :, :C], axis=2)
    rank = [2, 0, 3, 1]
    tb = oracle.table(L, y, K, C, tie=oracle.TIE_BEST_MEMBER, rank=rank)
    tl = oracle.table(L, y, K, C, tie=oracle.TIE_LOWEST_CLASS, rank=rank)
    for i in range(K):
        for j in range(i + 1, K):
            v = (1 << i) | (1 << j)
            better = i if rank[i] < rank[j] else j
            assert tb.cnt_vote[v - 1] == (top[:, better] == y).sum()
            both = ((top[:, i] == y) & (top[:, j] == y)).sum()
            dis = ((top[:, i] != top[:, j]) & (y == np.minimum(top[:, i], top[:, j]))).sum()
            assert tl.cnt_vote[v - 1] == both + dis


def test_I3_identical_models():
    C, N = 20, 300
    L1, y = _data(1, C, N, seed=5)
    L = np.repeat(L1, 3, axis=1)
    for tie in (0, 1):
        t = oracle.table(L, y, 3, C, tie=tie)
        assert len(set(t.cnt_vote.tolist())) == 1 and len(set(t.cnt_avg.tolist())) == 1
        assert t.cnt_vote[0] == t.cnt_avg[0]


def test_I4_full_set_average_is_mean_softmax():
    torch = pytest.importorskip("torch")
    K, C, N = 4, 50, 40
    L, y = _data(K, C, N, seed=6)
    v = (1 << K) - 1
    _, _, ap, _, _ = oracle.predict(L, K, C, v, want_avgprob=True)
    ref = torch.softmax(torch.tensor(L[:, :, :C], dtype=torch.float64), -1).mean(1).numpy()
    np.testing.assert_allclose(ap, ref, rtol=1e-13)


def test_I6_unanimous_samples_contribute_everywhere():
    K, C, N = 4, 10, 1500
    L, y = _data(K, C, N, seed=7)
    top = np.argmax(L[:, :, :C], axis=2)
    un = (top == top[:, :1]).all(1)
    assert un.sum() > 100
    t_un = oracle.table(L[un], y[un], K, C)
    want = int((top[un, 0] == y[un]).sum())
    assert (t_un.cnt_vote == want).all()
    # avg identity holds modulo oracle-flagged ambiguous pairs
    assert (np.abs(t_un.cnt_avg.astype(np.int64) - want) <= t_un.n_amb.astype(np.int64)).all()


def test_I7_model_permutation_permutes_mask_bits():
    K, C, N = 4, 12, 400
    L, y = _data(K, C, N, seed=8)
    rank = np.array([1, 3, 0, 2])
    perm = np.array([2, 0, 3, 1])  # new model i = old model perm[i]
    t0 = oracle.table(L, y, K, C, rank=rank)
    t1 = oracle.table(np.ascontiguousarray(L[:, perm, :]), y, K, C, rank=rank[perm])
    for v in range(1, 1 << K):
        old = sum(1 << int(perm[i]) for i in range(K) if (v >> i) & 1)
        assert t1.cnt_vote[v - 1] == t0.cnt_vote[old - 1]
        assert t1.cnt_avg[v - 1] == t0.cnt_avg[old - 1]


def test_I7_count_additivity_over_sample_partition():
    K, C, N = 3, 10, 900
    L, y = _data(K, C, N, seed=9)
    t = oracle.table(L, y, K, C)
    a = oracle.table(L[:317], y[:317], K, C)
    b = oracle.table(L[317:], y[317:], K, C)
    assert (t.cnt_vote == a.cnt_vote + b.cnt_vote).all()
    assert (t.cnt_avg == a.cnt_avg + b.cnt_avg).all()


def test_I8_no_monotonicity_enforced():
    # m0 always right; m1, m2 agree on the same wrong class on 2 of 3 samples.
    preds = np.array([[0, 1, 1], [1, 0, 0], [2, 2, 2]], np.int32)
    y = np.array([0, 1, 2], np.int32)
    t = oracle.table(onehot_logits(preds, 3), y, 3, 3)
    assert t.cnt_vote[0] == 3 and t.cnt_vote[6] == 1  # adding models lowered accuracy


def test_nonfinite_and_label_errors():
    L, y = _data(2, 5, 10)
    bad = L.copy(); bad[3, 1, 2] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.table(bad, y, 2, 5)
    assert e.value.code == oracle.ENONFINITE
    yy = y.copy(); yy[4] = 5
    with pytest.raises(oracle.OracleError) as e:
        oracle.table(L, yy, 2, 5)
    assert e.value.code == oracle.ELABEL
    ok = L.copy(); ok[3, 1, 2] = -np.inf  # -inf is a legal logit (probability 0)
    oracle.table(ok, y, 2, 5)


# ---------------------------------------------------------------- A1 heads (or_logits_gemm)
def _bf16_bits(vals):
    """bf16 bit patterns through torch's own float -> bfloat16 conversion (independent of gen/oracle)."""
    import torch
    t = torch.tensor(np.asarray(vals, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def _bf16_values(bits):
    """Exact widening through torch (bfloat16 -> float64), independent of the oracle's bit shifting."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()


def test_a1_hand_worked_example():
    """One row worked by hand: W indexing [m][c][d], scale 2^s applied to the dot only, then the bias."""
    rows = {r[0]: r[1:] for r in _read("a1_heads_example.txt")}
    s = int(rows["s"][0])
    X = _bf16_bits([[float(v) for v in rows["X"]]])
    W = _bf16_bits([[[float(v) for v in rows[f"W{m}{c}"]] for c in range(2)] for m in range(2)])
    b = np.array([float(v) for v in rows["bias"]], np.float32).reshape(2, 2)
    out = oracle.logits_gemm(X, W, b, s)
    assert out.reshape(-1).tolist() == [float(v) for v in rows["logits"]]
    # without bias: the scaled dots only
    assert oracle.logits_gemm(X, W, None, s).reshape(-1).tolist() == [1.25, -1.0, 0.125, -1.25]


@pytest.mark.parametrize("N,K,C,D,s", [(7, 3, 5, 64, -3), (5, 1, 2, 128, 0), (3, 4, 11, 192, 4)])
def test_a1_matches_einsum(N, K, C, D, s):
    """Random bf16 values with exponents in a narrow band (every product and partial sum exact in fp64, so
    the summation order cannot matter): the oracle equals numpy's einsum over torch-widened operands,
    scaled by an exact power of two, plus the bias. Non-square shapes catch transposed operands."""
    rng = np.random.default_rng(N * 131 + C)
    def vals(shape):
        return rng.choice([-1.0, 1.0], size=shape) * rng.integers(1, 256, size=shape) * 2.0 ** rng.integers(-8, 2, size=shape)
    X = _bf16_bits(vals((N, D)))
    W = _bf16_bits(vals((K, C, D)))
    b = (rng.integers(-64, 64, size=(K, C)) / 8.0).astype(np.float32)
    ref = np.einsum("nd,mcd->nmc", _bf16_values(X), _bf16_values(W)) * 2.0 ** s + b.astype(np.float64)[None]
    out = oracle.logits_gemm(X, W, b, s)
    assert out.shape == (N, K, C)
    np.testing.assert_array_equal(out, ref)
    # the generator's integer heads widen to small integers (integer-exact mode P3)
    psig, f0, df, sh = gen.head_params(D, C, K)
    Xg = gen.features(3, 0, N, D, C, psig, False)
    Wg = gen.weights(4, K, C, D, f0, df, False)
    ref_g = np.einsum("nd,mcd->nmc", _bf16_values(Xg), _bf16_values(Wg)) * 2.0 ** sh
    np.testing.assert_array_equal(oracle.logits_gemm(Xg, Wg, None, sh), ref_g)
