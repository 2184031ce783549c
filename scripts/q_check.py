"""Compare the labelled moments Q of the nested-batch kernel with the generic kernel (RK_Q_GENERIC)."""
import os, subprocess, sys, json
import numpy as np
if len(sys.argv) > 1:
    K, C, N, D = map(int, sys.argv[1:5])
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch, gen, paper_1804_06087_b200 as rk
    from bench import lat_profile
    B = [16, 32, 64, 128, 256]
    cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B), rates=[64.0, 128.0, 572.0, 1144.0])
    lab = torch.empty(N, dtype=torch.int32, device="cuda"); gen.dev_labels(1, 0, N, C, lab.data_ptr())
    psig, f0, df, sh = gen.head_params(D, C, K)
    X = torch.empty((N, D), dtype=torch.uint16, device="cuda")
    gen.dev_features(1, 0, N, D, C, psig, False, X.data_ptr(), lab.data_ptr())
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False), sh)
    ctx.score(X, N)
    t = ctx.subset_stats(lab, cfg)
    np.save(sys.argv[5], t["Q"])
else:
    for args in [("8", "1000", "1000000", "2048"), ("8", "1000", "250112", "2048"), ("12", "100", "300000", "1024")]:
        for mode in ("new", "generic"):
            env = dict(os.environ)
            if mode == "generic": env["RK_Q_GENERIC"] = "1"
            subprocess.check_call([sys.executable, __file__, *args, f"/tmp/q_{mode}.npy"], env=env)
        a, b = np.load("/tmp/q_new.npy"), np.load("/tmp/q_generic.npy")
        print(args, "equal" if np.array_equal(a, b) else f"DIFF {np.sum(a != b)} of {a.size}; new sum {a.sum()} generic {b.sum()}")
        print("  per (r, b) ratio new/generic:", np.round(a.sum(axis=2) / np.maximum(b.sum(axis=2), 1), 3).tolist())
