"""World-size-2 run of the library's NCCL all-reduce (A6) with both ranks on cuda:0 (the only GPU of a
gpurun box), if this NCCL build accepts two ranks on one device: each rank scores its lcm(B)-aligned shard
and rk_subset_finalize all-reduces the integer table; both ranks' tables must equal the one-rank table of
the whole batch. torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/nccl_two_ranks.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gen  # noqa: E402
import paper_1804_06087_b200 as rk  # noqa: E402
from bench import lat_profile  # noqa: E402
from paper_1804_06087_b200.shard import shard_ranges  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
K, C, D, N = 8, 1000, 256, 8192
B = [16, 32, 64, 128, 256]
cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B), rates=[128.0, 572.0])
psig, f0, df, sh = gen.head_params(D, C, K)
W, b = gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False)
off, n = shard_ranges(N, world, B)[rank]
buf = torch.zeros(128, dtype=torch.uint8)
if rank == 0:
    buf.copy_(torch.frombuffer(bytearray(rk.nccl_unique_id()), dtype=torch.uint8))
dist.broadcast(buf, 0)
ctx = rk.Context(0, rank, world, bytes(buf.numpy().tobytes()))
ctx.load_ensemble(K, C, D, W, b, sh)
y = torch.from_numpy(gen.labels(3, off, n, C)).cuda()
X = torch.from_numpy(gen.features(3, off, n, D, C, psig, False, y=gen.labels(3, off, n, C))).cuda()
ctx.score(X, n, off)
t = ctx.subset_stats(y, cfg)
ref = None
if rank == 0:
    one = rk.Context(0)
    one.load_ensemble(K, C, D, W, b, sh)
    ya = torch.from_numpy(gen.labels(3, 0, N, C)).cuda()
    Xa = torch.from_numpy(gen.features(3, 0, N, D, C, psig, False, y=gen.labels(3, 0, N, C))).cuda()
    one.score(Xa, N)
    ref = one.subset_stats(ya, cfg)
    for k in ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E"):
        assert np.array_equal(t[k], ref[k]), k
    assert t["N"] == N
tv = torch.from_numpy(t["cnt_vote"].astype(np.int64))
tl = [torch.zeros_like(tv) for _ in range(world)]
dist.all_gather(tl, tv)
assert all(torch.equal(tl[0], x) for x in tl)
print(f"rank {rank}: world-{world} NCCL table == one-rank table ({int(t['N'])} samples)", flush=True)
ctx.close()
dist.barrier()
dist.destroy_process_group()
