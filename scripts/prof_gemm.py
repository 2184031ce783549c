"""Time the head GEMM alone: python scripts/prof_gemm.py --K 8 --C 1000 --D 2048 --N 500000"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=8); ap.add_argument("--C", type=int, default=1000)
ap.add_argument("--D", type=int, default=2048); ap.add_argument("--N", type=int, default=500000)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
K, C, D, N = a.K, a.C, a.D, a.N
psig, f0, df, sh = gen.head_params(D, C, K)
lab = torch.empty(N, dtype=torch.int32, device="cuda")
X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
gen.dev_labels(1, 0, N, C, lab.data_ptr())
gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
ctx = rk.Context(0)
ctx.load_ensemble(K, C, D, gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False), sh)
ctx.score(X, N)
torch.cuda.synchronize()
ctx.set_profiling(True)
for _ in range(a.reps):
    ctx.score(X, N)
g = ctx.kernel_stats()["gemm_heads_tcgen05"]
print(f"gemm K={K} C={C} D={D} N={N}: {g['ms'] / g['launches']:.3f} ms, {g['flops'] / g['ms'] / 1e9:.0f} TFLOP/s")
