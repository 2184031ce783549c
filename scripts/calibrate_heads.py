#!/usr/bin/env python
"""Workload calibration of the synthetic dense heads against SURVEY.md §8(d)'s bands.

    python scripts/calibrate_heads.py --K 8 --C 1000 --D 2048 [--psig 5200 --f0 1000 --df 150 --sh -3]

Generates X, W, bias with gen/ (the bench's recipe), forms the logits in fp64 with numpy and prints the
ensemble statistics the bands are stated in: per-model top-1, unanimous fraction, mean max-softmax,
mean candidate set |S_c| (theta = min_j p[j][top_j] / K), full-set vote / average accuracy, and the
vote-stage worklist fraction (non-unanimous samples whose label is in S_c) with its mean |R|
(R = S_c ∩ {c : some model ranks c at or above y}). A development tool: not a test, not the oracle.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import gen  # noqa: E402


def stats(L, y):
    N, K, C = L.shape
    top = L.argmax(2)
    acc = (top == y[:, None]).mean(0)
    una = (top == top[:, :1]).all(1)
    P = np.exp(L - L.max(2, keepdims=True))
    P /= P.sum(2, keepdims=True)
    pmax = P.max(2)
    theta = pmax.min(1) / K
    Sc = (P >= theta[:, None, None]).any(1)  # [N][C]
    avg_acc = (P.mean(1).argmax(1) == y).mean()
    # full-set majority vote, lowest class on ties (a band statistic only)
    votes = np.zeros((N, C), np.int32)
    np.add.at(votes, (np.repeat(np.arange(N), K), top.ravel()), 1)
    vote_acc = (votes.argmax(1) == y).mean()
    y_in = Sc[np.arange(N), y]
    work = (~una) & y_in
    ly = L[np.arange(N), :, y]  # [N][K]
    above = (L >= ly[:, :, None]).any(1)  # [N][C]
    R = (Sc & above).sum(1) - 1
    return dict(acc=np.round(acc, 3).tolist(), unanimous=una.mean(), max_softmax=pmax.mean(),
                Sc_mean=Sc.sum(1).mean(), Sc_p99=np.percentile(Sc.sum(1), 99), vote_full=vote_acc, avg_full=avg_acc,
                gain=avg_acc - acc.max(), worklist=work.mean(), R_mean=R[work].mean() if work.any() else 0.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--C", type=int, default=1000)
    ap.add_argument("--D", type=int, default=2048)
    ap.add_argument("--N", type=int, default=3000)
    ap.add_argument("--psig", type=int)
    ap.add_argument("--f0", type=int)
    ap.add_argument("--df", type=int)
    ap.add_argument("--sh", type=int)
    ap.add_argument("--pnz", type=int, help="P(noise dim nonzero) * 65536 (0 = uniform {-1,0,1})")
    a = ap.parse_args()
    psig, f0, df, sh = gen.head_params(a.D, a.C, a.K)
    psig = a.psig if a.psig is not None else psig
    f0 = a.f0 if a.f0 is not None else f0
    df = a.df if a.df is not None else df
    sh = a.sh if a.sh is not None else sh
    if a.pnz is not None:
        psig = (psig & 0xffff) | (a.pnz << 16)
    y = gen.labels(1, 0, a.N, a.C)
    X = gen.bf16_to_f64(gen.features(1, 0, a.N, a.D, a.C, psig, False, y=y)).astype(np.float32)
    W = gen.bf16_to_f64(gen.weights(1000, a.K, a.C, a.D, f0, df, False)).astype(np.float32)
    b = gen.bias(2000, a.K, a.C, False).astype(np.float64)
    # integer products and sums stay below 2^24: the fp32 matmul is exact
    L = np.einsum("nd,mcd->nmc", X, W, optimize=True).astype(np.float64) * 2.0 ** sh + b[None]
    s = stats(L, y)
    print(f"psig={psig & 0xffff} pnz={psig >> 16} f0={f0} df={df} sh={sh}: " + ", ".join(
        f"{k}={v:.3f}" if isinstance(v, float) else f"{k}={v}" for k, v in s.items()))


if __name__ == "__main__":
    main()
