"""Vote-stage micro-run for profiling: rk_score_logits + rk_subset_stats on device-generated logits.

    python scripts/prof_vote.py --K 8 --C 1000 --N 200000 [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import lat_profile  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=8)
ap.add_argument("--C", type=int, default=1000)
ap.add_argument("--N", type=int, default=200_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tie", type=int, default=0)
ap.add_argument("--nocfg", action="store_true")
ap.add_argument("--gemm", type=int, default=0, help="D: feed the vote stage from the tcgen05 heads")
a = ap.parse_args()
K, C, N = a.K, a.C, a.N
ldc = (C + 3) // 4 * 4
lab = torch.empty(N, dtype=torch.int32, device="cuda")
L = torch.empty((N, K, ldc), dtype=torch.float32, device="cuda")
gen.dev_labels(1, 0, N, C, lab.data_ptr())
gen.dev_logits(1, 0, N, K, C, ldc, L.data_ptr(), lab.data_ptr())
B = [16, 32, 64, 128, 256]
cfg = None if a.nocfg else rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B),
                                         rates=[64.0, 128.0, 572.0, 1144.0])
ctx = rk.Context(0)
if a.gemm:  # vote stage fed by the tcgen05 heads (top1 / lse from the GEMM epilogue): bench path
    del L
    D = a.gemm
    psig, f0, df, sh = gen.head_params(D, C, K)
    X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
    gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
    ctx.load_ensemble(K, C, D, gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False), sh, tie=a.tie)
    ctx.score(X, N)
else:
    ctx.load_ensemble(K, C, tie=a.tie)
    ctx.score_logits(L, ldc, N)
torch.cuda.synchronize()
ctx.set_profiling(True)
for _ in range(a.reps):
    if a.gemm:
        ctx.score(X, N)
    t = ctx.subset_stats(lab, cfg)
ks = ctx.kernel_stats()
v = ks["vote_subsets"]
ms = v["ms"] / v["launches"]
print(f"K={K} C={C} N={N}: vote {ms:.3f} ms/launch, {v['bytes'] / v['launches'] / ms / 1e6:.1f} GB/s; "
      f"rechecks={int(t['n_recheck'].sum())} ({t['n_recheck'].sum() / N:.4f}/sample); "
      f"a(full)={t['cnt_vote'][-1] / N:.4f}")
for k, s in ks.items():
    if s["launches"]:
        print(f"  {k:22s} {s["ms"] / s["launches"]:.3f} ms x {s["launches"]}", (f"{s['flops'] / s['ms'] / 1e9:.0f} TFLOP/s" if s["flops"] else ""))
