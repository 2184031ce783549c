"""Per-repetition stage times of rk_subset_stats (GEMM-fed), to see run-to-run variance.

    python scripts/vote_reps.py K C N D REPS [v]

With a trailing "v" the heads are scored once and only rk_subset_stats repeats (no GEMM heating
between repetitions: A/B of vote-stage variants).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import lat_profile  # noqa: E402

K, C, N, D, R = map(int, sys.argv[1:6])
VOTE_ONLY = len(sys.argv) > 6 and sys.argv[6] == "v"
B = [16, 32, 64, 128, 256]
cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B), rates=[64.0, 128.0, 572.0, 1144.0])
lab = torch.empty(N, dtype=torch.int32, device="cuda")
gen.dev_labels(1, 0, N, C, lab.data_ptr())
psig, f0, df, sh = gen.head_params(D, C, K)
X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
ctx = rk.Context(0)
ctx.load_ensemble(K, C, D, gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False), sh)
ctx.set_profiling(True)
prev = {}
for i in range(R):
    if i == 0 or not VOTE_ONLY:
        ctx.score(X, N)
    t = ctx.subset_stats(lab, cfg)
    ks = ctx.kernel_stats()
    cur = {k: v["ms"] for k, v in ks.items()}
    print(i, " ".join(f"{k}={cur[k] - prev.get(k, 0):.3f}" for k in ("gemm_heads_tcgen05", "vote_subsets", "labelled_moments", "overdue_moments")),
          f"n_recheck={int(t['n_recheck'].sum())}")
    prev = cur
