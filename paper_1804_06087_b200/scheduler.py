"""NEXT-2: actor-critic training loop of the RL scheduler (§2.4, 426-436 §5.2).

Host orchestration only: every rollout, gradient and update runs in librk's kernels (csrc/rk_rl.cu,
rk_ac_rollout / rk_ac_grad / rk_ac_apply); this module owns the device buffers, draws the episodes'
start requests and reports per-iteration statistics of the trajectories.
"""
from __future__ import annotations

import numpy as np

from .rk import Context, RewardCfg


class ActorCritic:
    """Policy and value networks (one tanh hidden layer each, "a multi-layer perceptron") of
    the scheduler over the loaded ensemble's subsets x batch sizes, trained on episodes of the environment
    driven by `arrival` (device int64 [Narr] arrival times, e.g. from Context.sine_arrivals)."""

    def __init__(self, ctx: Context, cfg: RewardCfg, acc, arrival, L=16, H=64, n_steps=32, gamma=0.9,
                 reward_scale=None, seed=0, init_std=1.0, entropy=0.0):
        import torch
        self.torch = torch
        self.ctx, self.cfg = ctx, cfg
        self.acc = np.ascontiguousarray(acc, dtype=np.float64)
        self.arrival = arrival
        self.Narr = int(arrival.numel())
        self.B = np.asarray(cfg.B, np.int64)
        self.ac = {"L": L, "H": H, "n_steps": n_steps, "gamma": gamma,
                   "reward_scale": reward_scale if reward_scale is not None else 1.0 / float(max(cfg.B)),
                   "entropy": entropy}
        self.F, self.A, self.P = ctx.ac_dims(len(cfg.B), self.ac)
        F, A = self.F, self.A
        rng = np.random.default_rng(seed)
        parts = [rng.normal(0, init_std / np.sqrt(F), H * F), np.zeros(H),  # W1, b1
                 np.zeros(A * H), np.zeros(A),                              # W2, b2: uniform policy at start
                 rng.normal(0, init_std / np.sqrt(F), H * F), np.zeros(H),  # V1, c1
                 np.zeros(H), np.zeros(1)]                                  # v2, c2
        p = np.concatenate(parts).astype(np.float32)
        assert p.size == self.P
        self.params = torch.from_numpy(p).cuda()
        self.grad = torch.zeros_like(self.params)
        self.rng = np.random.default_rng(seed + 1)
        self.E = 0

    def buffers(self, E):
        t = self.torch
        n = self.ac["n_steps"]
        if self.E != E:
            self.traj = {"states": t.zeros((E, n, self.F), dtype=t.float32, device="cuda"),
                         "actions": t.zeros((E, n), dtype=t.int32, device="cuda"),
                         "rewards": t.zeros((E, n), dtype=t.float64, device="cuda"),
                         "overdue": t.zeros((E, n), dtype=t.int32, device="cuda")}
            self.E = E
        return self.traj

    def starts(self, E):
        span = self.Narr - self.ac["n_steps"] * int(self.B.max()) - 1
        if span < 1:
            raise ValueError("arrival array too short for n_steps batches of max(B)")
        return self.torch.from_numpy(self.rng.integers(0, span, E).astype(np.int64)).cuda()

    def rollout(self, E, seed, h0=None, forced=None):
        tr = self.buffers(E)
        h0 = self.starts(E) if h0 is None else h0
        self.ctx.ac_rollout(self.cfg, self.acc, self.arrival, self.Narr, self.ac, self.params, E, h0, tr,
                            forced=forced, seed=seed)
        return tr

    def stats(self, tr):
        """Per-episode return sum_t R_t (mean over episodes), accuracy sum a(v) b / sum b, overdue fraction."""
        t = self.torch
        a = tr["actions"].long()
        nB = len(self.B)
        b = t.as_tensor(self.B, device="cuda")[a % nB].double()
        accv = t.as_tensor(self.acc, device="cuda")[a // nB]
        return {"return": float(tr["rewards"].sum(1).mean()),
                "reward_per_request": float(tr["rewards"].sum() / b.sum()),
                "accuracy": float((accv * b).sum() / b.sum()),
                "overdue_frac": float(tr["overdue"].double().sum() / b.sum()),
                "mean_models": float(t.as_tensor([bin(v + 1).count("1") for v in range(len(self.acc))],
                                                 device="cuda", dtype=t.float64)[a // nB].mean())}

    def step(self, E, seed, lr_pi, lr_v):
        tr = self.rollout(E, seed)
        losses = self.ctx.ac_grad(self.cfg, self.ac, self.params, tr, E, self.grad)
        self.ctx.ac_apply(self.cfg, self.ac, self.params, self.grad, lr_pi, lr_v)
        s = self.stats(tr)
        s["loss_pi"], s["loss_v"] = float(losses[0]), float(losses[1])
        return s

    def train(self, iters, E=512, lr_pi=0.1, lr_v=0.1, seed0=0, log=None):
        curve = []
        for it in range(iters):
            s = self.step(E, seed0 + it, lr_pi, lr_v)
            s["iter"] = it
            curve.append(s)
            if log:
                log(s)
        return curve
