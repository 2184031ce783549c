"""Time rk_greedy_serve (NEXT-1, Algorithm 3 per rate and subset) at the c4 scale."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import CONFIGS, TAU_NS, BETA, lat_profile  # noqa: E402

for name in ("c4", "c5"):
    c = CONFIGS[name]
    K, N = c["K"], c["N"]
    ctx = rk.Context(0)
    ctx.load_ensemble(K, c["C"])
    cfg = rk.RewardCfg(B=c["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat_profile(K, c["B"]), rates=c["rates"])
    acc = np.full((1 << K) - 1, 0.8)
    r = ctx.greedy_serve(cfg, N, TAU_NS // 10, acc=acc)
    ctx.set_profiling(True)
    t0 = time.perf_counter()
    r = ctx.greedy_serve(cfg, N, TAU_NS // 10, acc=acc)
    wall = time.perf_counter() - t0
    ks = ctx.kernel_stats()["greedy_serve"]
    scen = len(c["rates"]) * ((1 << K) - 1)
    print(f"{name}: {scen} scenarios x {N} requests: kernel {ks['ms']:.2f} ms, call {wall * 1e3:.2f} ms, "
          f"{scen * N / (ks['ms'] / 1e3):.3e} request-decisions/s; overdue frac (full set, rates) "
          f"{(r['overdue'][:, -1] / N).round(3).tolist()}")
    ctx.close()
