"""N > 1 host path on CPU: two `gloo` ranks shard the request stream exactly like bench.py does
(boundaries at multiples of lcm(B), global arrival times), compute their shard's integer table with
the oracle, and sum it with a real all-reduce. The sum must equal the whole-dataset table bit-exactly
(invariant I7) — the property the library's single ncclAllReduce relies on."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

K, C, N = 3, 10, 1000
B = [16, 32, 48, 64]  # the paper's B, lcm 192 -> ragged last shard
KEYS = ("cnt_vote", "cnt_avg", "corr", "O", "Q", "E")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    import gen
    y = gen.labels(3, 0, N, C)
    L = gen.logits(3, 0, N, K, C, y=y)
    arr = np.cumsum(np.random.default_rng(1).integers(1, 30_000_000, N)).astype(np.int64)
    lat = np.array([[int(f * (16.67e6 + 3.333e6 * b)) for b in B] for f in (2.174, 1.679, 1.0)], np.int64)
    return y, L, arr, lat


def _worker(rank, world, port, out):
    import oracle
    from paper_1804_06087_b200.shard import shard_ranges
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    y, L, arr, lat = _inputs()
    off, n = shard_ranges(N, world, B)[rank]
    cfg = oracle.RewardCfg(B=B, beta=1.0, tau_ns=300_000_000, lat_ns=lat, arrival_ns=arr[off:off + n])
    t = oracle.table(L[off:off + n], y[off:off + n], K, C, cfg=cfg, threads=2)
    summed = {}
    for k in KEYS:
        ten = torch.from_numpy(getattr(t, k).astype(np.int64))
        dist.all_reduce(ten, op=dist.ReduceOp.SUM)
        summed[k] = ten.numpy()
    if rank == 0:
        out.put({k: v.tolist() for k, v in summed.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_table_equals_whole():
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y, L, arr, lat = _inputs()
    whole = oracle.table(L, y, K, C, cfg=oracle.RewardCfg(B=B, beta=1.0, tau_ns=300_000_000, lat_ns=lat,
                                                          arrival_ns=arr))
    for k in KEYS:
        np.testing.assert_array_equal(np.array(got[k]), getattr(whole, k).astype(np.int64), err_msg=k)


def test_shard_plan_matches_bench_layout():
    from paper_1804_06087_b200.shard import shard_ranges
    # c4 over 8 GPUs: boundaries at multiples of 256, last rank ragged
    rs = shard_ranges(1_000_000, 8, [16, 32, 64, 128, 256])
    assert all(off % 256 == 0 for off, _ in rs)
    assert sum(n for _, n in rs) == 1_000_000
    assert max(n for _, n in rs) - min(n for _, n in rs) <= 256
