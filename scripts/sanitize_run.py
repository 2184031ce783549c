"""Small drivers of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py c1|c2|k12|fused|serve|rl

Each run scores a small seeded batch through the C-ABI and checks the table against nothing (the parity
tests do that): the point is the sanitizer's verdict on the kernels' memory accesses and barriers."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import lat_profile  # noqa: E402

what = sys.argv[1]
SHAPES = {"c1": (3, 10, 1024, 1024), "c2": (3, 1000, 512, 1024), "k12": (12, 100, 256, 600), "fused": (8, 1000, 256, 768)}


def heads_ctx(K, C, D, N, tie=0):
    psig, f0, df, sh = gen.head_params(D, C, K)
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
    gen.dev_labels(5, 0, N, C, y.data_ptr())
    gen.dev_features(5, 0, N, D, C, psig, False, X.data_ptr(), y.data_ptr())
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, gen.weights(6, K, C, D, f0, df, False), gen.bias(7, K, C, False), sh, tie=tie)
    return ctx, X, y


B = [16, 32, 64]
if what in ("c1", "c2", "k12", "fused"):
    K, C, D, N = SHAPES[what]
    cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B), rates=[128.0, 572.0],
                       want_exceed=True, want_labelled=True)
    for tie in (0, 1):
        ctx, X, y = heads_ctx(K, C, D, N, tie)
        if what == "fused":
            ctx.score_labelled(X, y, N)
        else:
            ctx.score(X, N)
        t = ctx.subset_stats(y, cfg)
        print(what, tie, int(t["cnt_vote"][-1]), int(t["cnt_avg"][-1]))
        if what != "fused":
            pv = torch.zeros(N, dtype=torch.int32, device="cuda")
            ctx.predict((1 << K) - 1, pred_vote=pv, pred_avg=pv)
    if what == "k12":  # caller logits through the K >= 9 averaging kernels, queue mode
        L = torch.empty((N, K, 100), dtype=torch.float32, device="cuda")
        y = torch.empty(N, dtype=torch.int32, device="cuda")
        gen.dev_labels(9, 0, N, C, y.data_ptr())
        gen.dev_logits(9, 0, N, K, C, 100, L.data_ptr(), y.data_ptr())
        ctx = rk.Context(0)
        ctx.load_ensemble(K, C)
        ctx.score_logits(L, 100, N)
        cfg.queue = True
        ctx.subset_stats(y, cfg)
elif what == "serve":
    K, C, D, N = 3, 100, 256, 3000
    ctx, X, y = heads_ctx(K, C, D, N)
    arr = torch.empty(N, dtype=torch.int64, device="cuda")
    ctx.sine_arrivals(arr, N, 572.0, 500 * 560_000_000, 50_000_000, 0.1, 3)
    cfg = rk.RewardCfg(B=[16, 32, 48, 64], beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, [16, 32, 48, 64]),
                       arrival_ns=arr)
    ctx.greedy_serve(cfg, N, 0, acc=np.full(7, 0.8))
    ctx.async_serve(cfg, N, 0, acc=np.full(3, 0.8))
    pv = torch.zeros(N, dtype=torch.int32, device="cuda")
    print(ctx.serve_stream(X, N, cfg, 0, 7, pv, pv))
elif what == "rl":
    from paper_1804_06087_b200.scheduler import ActorCritic
    K = 3
    ctx = rk.Context(0)
    ctx.load_ensemble(K, 10)
    arr = torch.empty(50_000, dtype=torch.int64, device="cuda")
    ctx.sine_arrivals(arr, 50_000, 572.0, 500 * 560_000_000, 50_000_000, 0.1, 3)
    cfg = rk.RewardCfg(B=[16, 32, 48, 64], beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, [16, 32, 48, 64]),
                       rates=[1.0])
    ag = ActorCritic(ctx, cfg, np.full(7, 0.8), arr, L=8, H=32, n_steps=8)
    print(ag.train(2, E=16, lr_pi=0.5, lr_v=0.02)[-1]["return"])
torch.cuda.synchronize()
print("done", what)
