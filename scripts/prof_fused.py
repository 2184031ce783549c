"""One fused (NEXT-3) c4-shape step at a given N, for ncu: python scripts/prof_fused.py --N 262144 [--unfused]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import CONFIGS, BETA, TAU_NS, lat_profile  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=262144)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--unfused", action="store_true")
a = ap.parse_args()
c = CONFIGS["c4"]
K, C, D, N = c["K"], c["C"], c["D"], a.N
psig, f0, df, sh = gen.head_params(D, C, K)
lab = torch.empty(N, dtype=torch.int32, device="cuda")
X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
gen.dev_labels(1, 0, N, C, lab.data_ptr())
gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
ctx = rk.Context(0)
ctx.load_ensemble(K, C, D, gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False), sh)
cfg = rk.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat_profile(K, c["B"]), rates=c["rates"])
ctx.set_profiling(True)
for _ in range(a.reps):
    if a.unfused:
        ctx.score(X, N)
    else:
        ctx.score_labelled(X, lab, N)
    ctx.subset_stats(lab, cfg)
torch.cuda.synchronize()
ks = ctx.kernel_stats()
print({k: round(v["ms"] / max(1, v["launches"]), 3) for k, v in ks.items() if v["launches"]}, ctx.vote_diag())
