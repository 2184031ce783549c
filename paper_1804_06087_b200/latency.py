"""c(m, b) measured from this library's own kernels.

The paper's inference time of model m on a batch of b requests depends on "the model complexity,
hardware efficiency ... and the batch size". Here a model is one dense head, so c(m, b)
is the device time of serving one batch of b requests with model m alone: its head GEMM (`rk_score`,
tcgen05) followed by the per-request prediction of the action v = {m} (`rk_predict`). Each (m, b) runs
in its own one-model context and is timed with CUDA events around `reps` back-to-back batches on the
launching stream after warm-up; the median per batch is returned in integer nanoseconds, the unit of
`RewardCfg.lat_ns` (readings Q8-Q10). Nothing here computes the method: it only times the C-ABI calls.
"""
from __future__ import annotations

import numpy as np

from . import rk


def measure_lat_ns(W: np.ndarray, bias: np.ndarray | None, scale_log2: int, B, X, reps: int = 20,
                   warmup: int = 3, device: int = 0) -> np.ndarray:
    """W: bf16 bit patterns [K][C][D] (uint16); bias: [K][C] fp32 or None; X: a device uint16 tensor
    [>= max(B)][D] of features. Returns int64 [K][len(B)] with c(m, b) in ns."""
    import torch

    K, C, D = W.shape
    if X.shape[0] < max(B) or X.shape[1] != D:
        raise ValueError("X must hold at least max(B) rows of D features")
    out = np.zeros((K, len(B)), np.int64)
    stream = torch.cuda.current_stream()
    for m in range(K):
        ctx = rk.Context(device)
        ctx.load_ensemble(1, C, D, np.ascontiguousarray(W[m:m + 1]),
                          None if bias is None else np.ascontiguousarray(bias[m:m + 1]), scale_log2)
        pv = torch.empty(max(B), dtype=torch.int32, device="cuda")
        for bi, b in enumerate(B):
            for _ in range(warmup):
                ctx.score(X, b, 0, stream)
                ctx.predict(1, pv[:b], None, None, stream)
            times = []
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ctx.score(X, b, 0, stream)
                ctx.predict(1, pv[:b], None, None, stream)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            out[m, bi] = int(round(float(np.median(times)) * 1e6))
        ctx.close()
    return out
