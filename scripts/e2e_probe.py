"""e2e variants at c4 through the C-ABI with pinned host X and labels: one rk_score + rk_subset_stats per
step, or the step streamed in chunks (rk_subset_reset, rk_score + rk_subset_accumulate per chunk,
rk_subset_finalize). python scripts/e2e_probe.py [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import CONFIGS, BETA, TAU_NS, lat_profile  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = CONFIGS["c4"]
K, C, D, N = c["K"], c["C"], c["D"], c["N"]
psig, f0, df, sh = gen.head_params(D, C, K)
lab = torch.empty(N, dtype=torch.int32, device="cuda")
X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
gen.dev_labels(1, 0, N, C, lab.data_ptr())
gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
Xh = torch.empty((N, D), dtype=torch.uint16, pin_memory=True); Xh.copy_(X)
yh = torch.empty(N, dtype=torch.int32, pin_memory=True); yh.copy_(lab)
Xn, yn = Xh.numpy(), yh.numpy()
cfg = rk.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat_profile(K, c["B"]), rates=c["rates"],
                   want_exceed=True, want_labelled=True)
ctx = rk.Context(0)
ctx.load_ensemble(K, C, D, gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False), sh)
st = torch.cuda.current_stream()


def single():
    ctx.score(Xn, N, 0, st)
    return ctx.subset_stats(yn, cfg, st)


def streamed(ch):
    def f():
        ctx.subset_reset(cfg)
        for c0 in range(0, N, ch):
            m = min(ch, N - c0)
            ctx.score(Xn[c0:c0 + m], m, c0, st)
            ctx.subset_accumulate(yn[c0:c0 + m], st)
        return ctx.subset_finalize(st)
    return f


ref = None
for name, f in [("single", single), ("stream131k", streamed(131072)), ("stream262k", streamed(262144)),
                ("stream65k", streamed(65536)), ("single", single)]:
    t = f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        t = f()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    if ref is None:
        ref = t
    same = all((t[k] == ref[k]).all() for k in ("cnt_vote", "cnt_avg", "O", "Q", "E"))
    print(f"{name:12s} {ms:7.2f} ms  {N * ((1 << K) - 1) / ms * 1e3:.3e} sample·subset/s  table_equal={same}")
