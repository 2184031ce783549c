#!/usr/bin/env python
"""NEXT-2 experiment: train the actor-critic scheduler on the GPU for the
paper's trio setting (K = 3, B = {16, 32, 48, 64}, tau = 560 ms, beta = 1) under the
sine-plus-noise arrivals anchored at r_l = 128 and r_u = 572 req/s, with a(v) the
vote accuracies of every subset measured by this library on the c2-shape workload (K = 3, C = 1000,
50,000 samples). Compares, per request, with the paper's two baselines on the same arrival process:
synchronous full ensemble + Algorithm 3 (rk_greedy_serve, v = all) and asynchronous one model per batch
(rk_async_serve). Writes profiles/r02_scheduler.json.

    python scripts/train_scheduler.py [--iters 150] [--episodes 512]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import BETA, TAU_NS, lat_profile  # noqa: E402
from paper_1804_06087_b200.scheduler import ActorCritic  # noqa: E402


def subset_accuracy(ctx, K, C, D, N):
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
    gen.dev_labels(1, 0, N, C, y.data_ptr())
    gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), y.data_ptr())
    ctx.load_ensemble(K, C, D, W, b, sh)
    ctx.score(X, N)
    t = ctx.subset_stats(y)
    return t["cnt_vote"].astype(np.float64) / N


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1500)
    ap.add_argument("--episodes", type=int, default=512)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--lr-pi", type=float, default=1.0)
    ap.add_argument("--lr-v", type=float, default=0.02)
    ap.add_argument("--entropy", type=float, default=0.01, help="entropy bonus of the policy loss (PPO, X4)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_scheduler.json"))
    a = ap.parse_args()
    K, C, D, B = 3, 1000, 2048, [16, 32, 48, 64]
    ctx = rk.Context(0)
    acc = subset_accuracy(ctx, K, C, D, 50_000)
    lat = lat_profile(K, B)
    N = 2_000_000
    period = 500 * TAU_NS
    res = {"K": K, "B": B, "tau_ns": TAU_NS, "beta": BETA, "acc": acc.tolist(), "lat_ns": lat.tolist(),
           "learner": {"lr_pi": a.lr_pi, "lr_v": a.lr_v, "entropy": a.entropy, "episodes": a.episodes, "steps": a.steps},
           "arrivals": {"process": "sine + noise (reading Q16)", "period_ns": period, "delta_ns": 50_000_000,
                        "noise_std": 0.1}, "runs": {}}
    for name, ref in (("r_l", 128.0), ("r_u", 572.0)):
        arr = torch.empty(N, dtype=torch.int64, device="cuda")
        ctx.sine_arrivals(arr, N, ref, period, 50_000_000, 0.1, 7)
        cfg = rk.RewardCfg(B=B, beta=BETA, tau_ns=TAU_NS, lat_ns=lat, arrival_ns=arr)
        # baselines on the whole stream (per request)
        sync = ctx.greedy_serve(cfg, N, 0, acc=acc)
        full = (1 << K) - 2
        asy = ctx.async_serve(cfg, N, 0, acc=acc[[0, 1, 3]])  # a({m}) for m = 0, 1, 2 (v = 1, 2, 4)
        base = {
            "sync_full_ensemble": {"reward_per_request": float(sync["reward"][0, full] / max(1, sync["served"][0, full])),
                                   "overdue_frac": float(sync["overdue"][0, full] / max(1, sync["served"][0, full])),
                                   "accuracy": float(acc[full])},
            "async_one_model": {"reward_per_request": float(asy["reward"][0] / max(1, asy["served"][0])),
                                "overdue_frac": float(asy["overdue"][0] / max(1, asy["served"][0])),
                                "batches_per_model": asy["model_batches"][0].tolist()},
        }
        torch.manual_seed(0)
        agent = ActorCritic(ctx, cfg, acc, arr, L=16, H=64, n_steps=a.steps, seed=0, entropy=a.entropy)
        t0 = time.perf_counter()
        curve = agent.train(a.iters, E=a.episodes, lr_pi=a.lr_pi, lr_v=a.lr_v,
                            log=lambda s: print(name, s["iter"], round(s["return"], 2), round(s["overdue_frac"], 3),
                                                round(s["accuracy"], 4), round(s["mean_models"], 2), flush=True))
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        last = curve[-10:]
        served = a.episodes * a.steps
        res["runs"][name] = {
            "ref_rate": ref, "iters": a.iters, "episodes_per_iter": a.episodes, "steps": a.steps,
            "train_s": el, "decisions_per_s": a.iters * served / el,
            "curve": [{k: c[k] for k in ("iter", "return", "reward_per_request", "accuracy", "overdue_frac", "mean_models", "loss_pi",
                                         "loss_v")} for c in curve],
            "final": {k: float(np.mean([c[k] for c in last])) for k in ("return", "reward_per_request", "accuracy",
                                                                        "overdue_frac", "mean_models")},
            "baselines": base}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps({k: v["final"] for k, v in res["runs"].items()}))


if __name__ == "__main__":
    main()
