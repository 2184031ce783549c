"""N > 1 with the library itself ("a 2-rank test that drives librk ... with the NCCL path
mocked"): two processes on the one GPU of a test box each run librk's whole path on its lcm(B)-aligned
shard with its global offset (bench.py's layout), and the integer tables are summed by a
gloo all-reduce standing in for the library's ncclAllReduce (NCCL refuses two ranks on one device,
profiles/r02_nccl_two_ranks_one_gpu.log). The sum must equal the one-process table of the whole batch and
the oracle's, bit-exactly, including the rate-driven overdue / labelled moments that depend on the
offset."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

K, C, D, N = 8, 1000, 256, 6000
B = [16, 32, 64, 128, 256]
RATES = [64.0, 572.0]
KEYS = ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _heads():
    import gen
    psig, f0, df, sh = gen.head_params(D, C, K)
    W, b = gen.weights(1000, K, C, D, f0, df, False), gen.bias(2000, K, C, False)
    return psig, W, b, sh


def _cfg(rk):
    from gpu_helpers import lat_profile
    return rk.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(K, B), rates=RATES)


def _worker(rank, world, port, out):
    import gen
    import paper_1804_06087_b200 as rk
    from paper_1804_06087_b200.shard import shard_ranges
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    psig, W, b, sh = _heads()
    off, n = shard_ranges(N, world, B)[rank]
    y = gen.labels(4, off, n, C)
    X = gen.features(4, off, n, D, C, psig, False, y=y)
    ctx = rk.Context(0)
    ctx.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh)
    ctx.score(torch.from_numpy(X).cuda(), n, off)
    t = ctx.subset_stats(torch.from_numpy(y).cuda(), _cfg(rk))
    summed = {}
    for k in KEYS + ("N",):
        ten = torch.from_numpy(np.asarray(t[k]).astype(np.int64).reshape(-1))
        dist.all_reduce(ten, op=dist.ReduceOp.SUM)
        summed[k] = ten.numpy().tolist()
    if rank == 0:
        out.put(summed)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_librk_tables_sum_to_whole():
    import gen
    import oracle
    import paper_1804_06087_b200 as rk
    from gpu_helpers import compare_tables, default_cfg
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    psig, W, b, sh = _heads()
    y = gen.labels(4, 0, N, C)
    X = gen.features(4, 0, N, D, C, psig, False, y=y)
    one = rk.Context(0)
    one.load_ensemble(K, C, D, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), sh)
    one.score(torch.from_numpy(X).cuda(), N)
    whole = one.subset_stats(torch.from_numpy(y).cuda(), _cfg(rk))
    assert got["N"][0] == N
    for k in KEYS:
        np.testing.assert_array_equal(np.array(got[k]), np.asarray(whole[k]).astype(np.int64).reshape(-1), err_msg=k)
    _, ocfg = default_cfg(K, B=B, rates=RATES)
    o = oracle.table(oracle.logits_gemm(X, W, b, sh), y, K, C, cfg=ocfg)
    compare_tables(whole, o, K=K)
    one.close()
