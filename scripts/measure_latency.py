"""NEXT-1: print c(m, b) measured from this library's kernels for a bench config (int64 ns, [K][nB]),
next to the paper-line profile bench.py uses.

    python scripts/measure_latency.py --config c4
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
from bench import CONFIGS, lat_profile  # noqa: E402
from paper_1804_06087_b200.latency import measure_lat_ns  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
cfg = CONFIGS[a.config]
K, C, D, B = cfg["K"], cfg["C"], cfg["D"], cfg["B"]
psig, f0, df, sh = gen.head_params(D, C, K)
W = gen.weights(1000, K, C, D, f0, df, False)
b = gen.bias(2000, K, C, False)
X = torch.empty((max(B), D), dtype=torch.uint16, device="cuda")
lab = torch.empty(max(B), dtype=torch.int32, device="cuda")
gen.dev_labels(1, 0, max(B), C, lab.data_ptr())
gen.dev_features(1, 0, max(B), D, C, psig, False, X.data_ptr(), lab.data_ptr())
lat = measure_lat_ns(W, b, sh, B, X, reps=a.reps)
print(f"{a.config}: K={K} C={C} D={D} B={B}")
print("measured c(m,b) [us]:")
for m in range(K):
    print(f"  m={m}: " + " ".join(f"{x / 1e3:8.1f}" for x in lat[m]))
print("paper-line profile (bench.py) [ms]: " + " ".join(f"{x / 1e6:.1f}" for x in lat_profile(K, B)[0]))
