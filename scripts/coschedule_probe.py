"""Probe: does the vote stage co-run with the head GEMM on the same SMs?

Context A scores half the c4 samples (GEMM) on stream s1 while context B runs rk_subset_stats on the
other half (already scored) on stream s2; compares against running the two back to back.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import lat_profile  # noqa: E402

K, C, D, N = 8, 1000, 2048, 499_968  # multiple of lcm(B) = 256
psig, f0, df, sh = gen.head_params(D, C, K)
W = gen.weights(1000, K, C, D, f0, df, False)
b = gen.bias(2000, K, C, False)
lab = torch.empty(2 * N, dtype=torch.int32, device="cuda")
X = torch.empty((2 * N, D), dtype=torch.uint16, device="cuda")
gen.dev_labels(1, 0, 2 * N, C, lab.data_ptr())
gen.dev_features(1, 0, 2 * N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
B = [16, 32, 64, 128, 256]
cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B), rates=[64.0, 128.0, 572.0, 1144.0])
A, Bc = rk.Context(0), rk.Context(0)
for c in (A, Bc):
    c.load_ensemble(K, C, D, W, b, sh)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
Bc.score(X[N:], N, N, s2)
torch.cuda.synchronize()


def seq():
    A.score(X[:N], N, 0, s1)
    torch.cuda.synchronize()
    Bc.subset_stats(lab[N:], cfg, s2)
    torch.cuda.synchronize()


def par():
    A.score(X[:N], N, 0, s1)        # async on s1
    Bc.subset_stats(lab[N:], cfg, s2)  # vote kernels on s2 while the GEMM runs; returns after its D2H
    torch.cuda.synchronize()


for f in (seq, par, seq, par):
    f()
A.set_profiling(True)
Bc.set_profiling(True)


def kstats():
    a, b = A.kernel_stats(), Bc.kernel_stats()
    return a.get("gemm_heads_tcgen05", {}).get("ms", 0.0), b.get("vote_subsets", {}).get("ms", 0.0)


for name, f in (("sequential", seq), ("concurrent", par)):
    g0, v0 = kstats()
    t0 = time.perf_counter()
    for _ in range(5):
        f()
    g1, v1 = kstats()
    print(f"{name}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms  (gemm events {(g1 - g0) / 5:.2f} ms, "
          f"vote events {(v1 - v0) / 5:.2f} ms)")
A.score(X[:N], N, 0, s1); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    A.score(X[:N], N, 0, s1)
torch.cuda.synchronize()
print(f"gemm alone: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms")
t0 = time.perf_counter()
for _ in range(5):
    Bc.subset_stats(lab[N:], cfg, s2)
torch.cuda.synchronize()
print(f"vote alone: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms")
