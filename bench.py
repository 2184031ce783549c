#!/usr/bin/env python
"""Benchmark of the hot path: X -> K tcgen05 heads -> vote / average over all 2^K-1 subsets ->
per-(subset, batch) counts and batch moments -> [NCCL all-reduce] -> reward table.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl rk|reference]

One JSON line (rank 0). Metric (BASELINE.json): sample·subset evaluations per second = N_total * S
per step / step time (max over ranks, CUDA events). Inputs are synthetic, seeded, generated in HBM
before the timed region (X is 4 GB at c4 >> 126 MB L2, so no L2 flush is needed between steps).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sample·subset evaluations/sec at 1/2/4/8 B200; vote-stage HBM GB/s vs peak"
UNIT = "sample·subset/s"

# BASELINE.json configs as concrete runs; D is our choice (the paper has no heads).
CONFIGS = {
    "c1": dict(K=3, C=10, N=1_000, D=1024, B=[16, 32, 64], rates=[64.0, 128.0, 572.0, 1144.0]),
    "c2": dict(K=3, C=1000, N=50_000, D=2048, B=[16, 32, 48, 64], rates=[128.0, 572.0]),
    "c3": dict(K=6, C=1000, N=1_000_000, D=2048, B=[16, 32, 64, 128, 256], rates=[64.0, 128.0, 572.0, 1144.0]),
    "c4": dict(K=8, C=1000, N=1_000_000, D=2048, B=[16, 32, 64, 128, 256], rates=[64.0, 128.0, 572.0, 1144.0]),
    "c5": dict(K=12, C=100, N=4_000_000, D=1024, B=[16, 32, 64, 128, 256], rates=[64.0, 128.0, 572.0, 1144.0]),
}
TAU_NS = 560_000_000  # PAPER.md:700 (printed value; X3)
BETA = 1.0


def lat_profile(K, B):
    """c(m,b) = f_m * (16.67 ms + 3.333 ms * b): the line through the paper's c(16)=70 ms, c(64)=230 ms
    (PAPER.md:700); K=3 uses the trio factors reproducing r_u=572, r_l=128."""
    f = [2.174, 1.679, 1.000] if K == 3 else [1.6 - 0.1 * m for m in range(K)]
    return np.array([[int(round(f[m] * (16.67e6 + 3.333e6 * b))) for b in B] for m in range(K)], np.int64)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(cfgname, cfg, budget_s=15.0):
    """The CPU oracle as it stands, on a bounded sample of the same workload (rank 0, N=1 only)."""
    import gen
    import oracle
    K, C, D = cfg["K"], cfg["C"], cfg["D"]
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    lat = lat_profile(K, cfg["B"])
    ocfg = oracle.RewardCfg(B=cfg["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat, rates=cfg["rates"], want_exceed=True)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    L = 1
    from math import gcd
    for bb in cfg["B"]:
        L = L * bb // gcd(L, bb)
    n = L
    total_t, total_n = 0.0, 0
    while True:
        y = gen.labels(1, total_n, n, C)
        X = gen.features(1, total_n, n, D, C, psig, False, y=y)
        t0 = time.perf_counter()
        lg = oracle.logits_gemm(X, W, b, sh)
        oracle.table(lg, y, K, C, cfg=ocfg, threads=cores)
        dt = time.perf_counter() - t0
        total_t += dt
        total_n += n
        if total_t > budget_s * 0.5 or total_n >= cfg["N"]:
            break
        n = min(cfg["N"] - total_n, max(L, int(n * max(1.0, (budget_s * 0.5 - total_t) / max(dt, 1e-3))) // L * L))
    S = (1 << K) - 1
    return {"value": total_n * S / total_t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {total_n} samples of {cfgname} (full hot path: fp64 heads + all {S} subsets + moments), "
                      f"{total_t:.1f} s on {cores} host threads"}


def reference_arm(args, cfgname, cfg, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    K = cfg["K"]
    S = (1 << K) - 1
    per_step_budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    base = cpu_baseline(cfgname, cfg, budget_s=per_step_budget * 2)
    # steps: repeat bounded samples; the oracle's throughput is stable, report the measured one
    times, secs = [], []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        b = cpu_baseline(cfgname, cfg, budget_s=per_step_budget * 2)
        secs.append(time.perf_counter() - t0)
        times.append(b["value"])
    val = statistics.median(times)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": cfg["N"] * S / val * 1e3,
            "ms_per_step_kind": "extrapolated: the full workload's N*S divided by the measured oracle RATE; each "
                                "timed step is a bounded sample (sample_ms_per_step)",
            "sample_ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfgname, **{k: cfg[k] for k in ("K", "C", "N", "D", "B")}},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": base["cores"], "kind": "oracle", "sample": base["sample"]},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_stats(ctx, labels, K, C, nsamp=4096):
    """Statistics of the benchmarked workload (reporting only, outside the timed region): from the first
    nsamp rows' logits (rk_outputs) in fp64 numpy -- unanimous fraction, mean number of distinct member
    predictions d, mean candidate set |S_c| (theta = min_j p[j][top_j] / K), and on the
    non-unanimous samples whose label is in S_c (the averaging worklist) the mean |R|, R = S_c ∩ {c != y :
    some model has l[m][c] >= l[m][y]}."""
    import torch
    out = ctx.outputs()
    if not out["logits"]:
        return {}
    ldc = out["ldc"]
    ns = min(nsamp, out["N"])

    class _View:  # the library's logits workspace as a torch view (no copy on the device)
        __cuda_array_interface__ = {"shape": (ns, K, ldc), "typestr": "<f4", "data": (out["logits"], False),
                                    "version": 3}

    torch.cuda.synchronize()
    L = torch.as_tensor(_View(), device="cuda")[:, :, :C].double().cpu().numpy()
    y = labels[:ns].cpu().numpy()
    top = L.argmax(2)
    una = (top == top[:, :1]).all(1)
    d = np.array([len(set(r)) for r in top])
    P = np.exp(L - L.max(2, keepdims=True))
    P /= P.sum(2, keepdims=True)
    theta = P.max(2).min(1) / K
    Sc = (P >= theta[:, None, None]).any(1)
    ly = L[np.arange(ns), :, y]
    above = (L >= ly[:, :, None]).any(1)
    R = (Sc & above).sum(1) - 1
    work = (~una) & Sc[np.arange(ns), y]
    return {"sample_rows": int(ns), "unanimous_frac": float(una.mean()), "mean_distinct_predictions": float(d.mean()),
            "mean_Sc": float(Sc.sum(1).mean()), "worklist_frac_sample": float(work.mean()),
            "mean_R_on_worklist": float(R[work].mean()) if work.any() else 0.0,
            "mean_d_nonunanimous": float(d[~una].mean()) if (~una).any() else 0.0,
            "mean_Sc_nonunanimous": float(Sc.sum(1)[~una].mean()) if (~una).any() else 0.0}


def kernels_per_step(K, C, cfg, queue, fused=False, fallback=True):
    """Our kernel launches in one step (rk_score + rk_subset_stats), mirroring the library's dispatch
    (csrc/rk_api.cpp, rk_vote_batch.cu); cross-checked against the ncu launch list in profiles/."""
    ldc = (C + 3) // 4 * 4
    n = 1  # gemm_heads_kernel
    if fused and K <= 8 and (C + 15) // 16 * 16 > 128:
        n += 2  # vote_classify_kernel + vote_sparse_average_kernel
        if fallback:
            n += 3  # gather_rows_kernel + gemm_heads_kernel + vote_average_kernel on the recomputed rows
    elif K <= 8:
        n += 2  # vote_classify_kernel + vote_average_kernel
    else:
        n += 1  # vote_group_classify_kernel
        if ldc <= 128:
            n += (2 if K == 12 else 1) + 1  # vote_wsample_average_kernel pass(es) + vote_pair_recheck_kernel
        n += 2  # vote_cta_average_kernel + vote_batch_average_kernel
    labelled = bool(cfg["B"]) and bool(cfg["rates"])
    if labelled:
        n += 1 + (1 if queue else 0)  # overdue_kernel (+ queue_scan_kernel)
    n += 1  # merge_kernel
    if labelled:
        n += 1  # q_nested_kernel / q_kernel
    n += 1  # fold_kernel
    return n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="rk", choices=["rk", "reference"])
    ap.add_argument("--tie", default="best_member", choices=["best_member", "lowest_class"])
    ap.add_argument("--queue", action="store_true", help="queue-aware latency (reading Q15, PAPER.md:410)")
    ap.add_argument("--fused", action="store_true",
                    help="NEXT-3 fused forward + vote (rk_score_labelled) instead of rk_score + the logits vote stage "
                         "(about 1.2 ms slower per c4 step on B200: DESIGN.md §6)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfgname = args.config
    cfg = CONFIGS[cfgname]
    if args.impl == "reference":
        reference_arm(args, cfgname, cfg, rank, world)
        return

    import torch
    import gen
    import paper_1804_06087_b200 as rk
    from paper_1804_06087_b200.shard import shard_ranges

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K, C, D, Ntot = cfg["K"], cfg["C"], cfg["D"], cfg["N"]
    S = (1 << K) - 1
    off, n = shard_ranges(Ntot, world, cfg["B"])[rank]
    # NCCL bootstrap for the library's own communicator (A6): rank 0 id, broadcast via torch.distributed
    nid = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(rk.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tobytes())
    ctx = rk.Context(local, rank, world, nid)
    psig, f0, df, sh = gen.head_params(D, C, K)
    W = gen.weights(1000, K, C, D, f0, df, False)
    b = gen.bias(2000, K, C, False)
    tie = rk.TIE_BEST_MEMBER if args.tie == "best_member" else rk.TIE_LOWEST_CLASS
    ctx.load_ensemble(K, C, D, W, b, sh, tie=tie)
    stream = torch.cuda.current_stream()
    labels = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    X = torch.empty((max(n, 1), D), dtype=torch.uint16, device="cuda")
    gen.dev_labels(1, off, n, C, labels.data_ptr(), stream.cuda_stream)
    gen.dev_features(1, off, n, D, C, psig, False, X.data_ptr(), labels.data_ptr(), stream.cuda_stream)
    lat = lat_profile(K, cfg["B"])
    rcfg = rk.RewardCfg(B=cfg["B"], beta=BETA, tau_ns=TAU_NS, lat_ns=lat, rates=cfg["rates"], want_exceed=True,
                        want_labelled=True, queue=args.queue)
    torch.cuda.synchronize()

    fused = args.fused

    def score(Xb, yb):
        if fused:
            ctx.score_labelled(Xb, yb, n, off, stream)  # NEXT-3: no logits stored for K <= 8, C > 128
        else:
            ctx.score(Xb, n, off, stream)

    def step():
        score(X, labels)
        return ctx.subset_stats(labels, rcfg, stream)

    for _ in range(max(3, args.warmup)):
        t = step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ctx.set_profiling(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # per-step boundaries for the median / min / max of SURVEY.md §8(d) (value uses the whole region)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    marks[0].record(stream)
    for i in range(args.steps):
        t = step()
        marks[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    per_step = sorted(marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps))
    ks = ctx.kernel_stats()
    diag = ctx.vote_diag() if K <= 8 else (0, 0, 0)
    ctx.set_profiling(False)
    clk = clocks.stop()
    if dist:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = Ntot * S / (ms_step / 1e3)

    # ---- e2e: through the C-ABI with HOST buffers (H2D of X and labels, D2H of the table, every step)
    Xh = torch.empty((max(n, 1), D), dtype=torch.uint16, pin_memory=True)
    yh = torch.empty(max(n, 1), dtype=torch.int32, pin_memory=True)
    Xh.copy_(X)
    yh.copy_(labels)
    Xh_np, yh_np = Xh.numpy(), yh.numpy()
    score(Xh_np, yh_np)
    ctx.subset_stats(yh_np, rcfg, stream)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        score(Xh_np, yh_np)
        ctx.subset_stats(yh_np, rcfg, stream)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if dist:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    # the e2e path's own ceiling: a plain pinned host->device copy of the same features (cudaMemcpyAsync),
    # device-timed, on this box
    hp0, hp1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    X.copy_(Xh, non_blocking=True)
    hp0.record(stream)
    for _ in range(2):
        X.copy_(Xh, non_blocking=True)
    hp1.record(stream)
    torch.cuda.synchronize()
    h2d_peak = 2 * n * D * 2 / (hp0.elapsed_time(hp1) / 1e3) / 1e9
    nB, nR = len(cfg["B"]), len(cfg["rates"])
    d2h = 8 * (4 + 3 * S + nB * S + 3 * nR * nB * S) + 16 * nR * nB * S

    peaks, peak_src = load_peaks()
    g = ks["gemm_heads_tcgen05"]
    v = ks["vote_subsets"]
    gemm_ms = g["ms"] / max(1, g["launches"])
    gemm_flops = g["flops"] / max(1, g["launches"])
    vote_ms = v["ms"] / max(1, v["launches"])
    vote_bytes = v["bytes"] / max(1, v["launches"])
    gemm_tfs = gemm_flops / (gemm_ms / 1e3) / 1e12
    vote_gbs = vote_bytes / (vote_ms / 1e3) / 1e9
    # Denominator: the measured BURST cuBLAS bf16 figure, always. The sustained one was measured over a
    # 4 s back-to-back loop at ~1.34 GHz under the power cap; a bench step alternates tensor-bound and
    # memory-bound kernels and its timed region is far shorter, so the clock stays well above that
    # regime (see `clocks`). The burst figure is the larger, i.e. conservative, denominator.
    peak_key = "bf16_tflops"
    peak_t = peaks.get(peak_key, peaks.get("bf16_tflops_sustained"))
    traffic = vtraffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):  # ncu dram bytes per launch of this workload (scripts/summarize_profiles.py)
        # the fused path (NEXT-3) moves different bytes: only its own capture's figures apply
        tj = json.load(open(tp)).get(cfgname + ("_fused" if fused else ""), {})
        traffic, vtraffic = tj.get("gemm_heads_tcgen05"), tj.get("vote_subsets")
    launches = args.steps * kernels_per_step(K, C, cfg, args.queue, fused, diag[1] > 0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "step_ms": {"median": per_step[len(per_step) // 2], "min": per_step[0], "max": per_step[-1], "rank": rank},
        "config": {"workload": cfgname, "K": K, "C": C, "N": Ntot, "D": D, "B": cfg["B"], "rates": cfg["rates"],
                   "tie": args.tie, "queue": bool(args.queue), "subsets": S,
                   "fused_forward_vote": bool(fused and K <= 8 and C > 128), "parallelism": f"samples sharded over {world} GPU(s)",
                   "l2": "inputs larger than L2 (X %.1f GB, logits %.1f GB)" % (Ntot * D * 2 / 1e9, Ntot * K * C * 4 / 1e9)},
        "roofline": {"bound": "tensor", "kernel": "gemm_heads_tcgen05", "achieved": gemm_tfs,
                     "peak": peak_t, "unit": "TFLOP/s", "frac": gemm_tfs / peak_t, "traffic": traffic,
                     "share_of_step": gemm_ms / ms_step,
                     "peak_source": f"{peak_src} {peak_key} (burst cuBLAS bf16; conservative, see DESIGN.md §9)",
                     "algorithmic": "2*D*K*C flop per sample"},
        "vote_stage": {"bound": "hbm", "kernel": "vote_subsets", "achieved": vote_gbs, "peak": peaks["hbm_gbs"],
                       "unit": "GB/s", "frac": vote_gbs / peaks["hbm_gbs"], "traffic": vtraffic,
                       "ms_per_launch": vote_ms,
                       "share_of_step": vote_ms / ms_step,
                       "algorithmic": "(K*C*4 + 4) bytes per sample"},
        "kernels_ms_per_step": {k: ks[k]["ms"] / args.steps for k in ks if ks[k]["launches"]},
        "e2e": {"value": Ntot * S / e2e_s, "unit": UNIT, "h2d_bytes_per_step": n * D * 2 + n * 4,
                "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "ms_per_step": e2e_s * 1e3,
                # the bound of this path: the host->device copy of the features over PCIe (pinned source)
                "h2d_gbs": (n * D * 2 + n * 4) / e2e_s / 1e9, "bound": "pcie h2d",
                "h2d_peak_gbs": h2d_peak, "frac": (n * D * 2 + n * 4) / e2e_s / 1e9 / h2d_peak},
        "gpu_launches": launches,
        "clocks": clk,
        "rank0_check": {"N": int(t["N"]), "a_full_set": float(t["cnt_vote"][-1]) / max(1, int(t["N"])),
                        "a_best_single": float(t["cnt_vote"][0]) / max(1, int(t["N"]))},
    }
    if K <= 8:
        wl, fb, sk = diag
        line["vote_stage"]["worklist_frac"] = wl / max(1, n)
        line["vote_stage"]["fallback_frac"] = fb / max(1, n)
        # rows of worklist samples the averaging kernel did not stream (second-largest-logit proof)
        line["vote_stage"]["rows_skipped_frac"] = sk / max(1, wl * K)
    ws = workload_stats(ctx, labels, K, C) if rank == 0 and not fused else {}
    line["workload_stats"] = ws
    if vtraffic:  # the honest figure: ncu DRAM bytes of this workload's vote stage per launch / its time
        line["vote_stage"]["dram_bytes_per_launch"] = vtraffic
        line["vote_stage"]["achieved_dram"] = vtraffic / (vote_ms / 1e3) / 1e9
        line["vote_stage"]["frac_dram"] = line["vote_stage"]["achieved_dram"] / peaks["hbm_gbs"]
    if vote_ms > gemm_ms and ws:  # the vote stage dominates (K >= 9): an ALU-bound roofline kernel
        # SURVEY.md §8(d)'s algorithmic op count: K*C argmax compares + K*C exp per sample, plus on the
        # non-unanimous samples S * (d + |S_c| + 2) (a vote tally over the d distinct predictions, an
        # average over the candidate set, a compare and a count per subset); d and |S_c| are this
        # workload's means (workload_stats). Peak: 148 SMs x 128 int32/fp32 lanes x the SM clock
        # (B200_PROFILING.md unit counts).
        sm_mhz = clk.get("sm_max_mhz") or 1965.0
        nonu = 1.0 - ws["unanimous_frac"]
        per_sample = 2.0 * K * C + nonu * S * (ws["mean_d_nonunanimous"] + ws["mean_Sc_nonunanimous"] + 2.0)
        ops = n * per_sample
        alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e9
        alu = ops / (vote_ms / 1e3) / 1e9
        line["gemm_stage"] = line["roofline"]
        line["roofline"] = {"bound": "alu", "kernel": "vote_subsets", "achieved": alu, "peak": alu_peak,
                            "unit": "Gop/s", "frac": alu / alu_peak, "traffic": vtraffic,
                            "share_of_step": vote_ms / ms_step,
                            "peak_source": f"148 SMs x 128 lanes x {sm_mhz:.0f} MHz (B200 unit counts)",
                            "algorithmic": "2*K*C + (1 - unanimous) * S * (d + |S_c| + 2) ops per sample "
                                           f"(SURVEY.md §8(d); {per_sample:.0f} here)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfgname, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
