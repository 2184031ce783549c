"""Pins of the asynchronous one-model-per-batch baseline (NEXT-1; reading S2): two
hand-worked traces, and invariants -- with one model it is Algorithm 3 itself (the synchronous policy of
the singleton subset), and every request is served or left unserved."""
import os

import numpy as np

import oracle
from bench import lat_profile

GOLD = os.path.join(os.path.dirname(__file__), "golden", "s2_async_serve.txt")


def gold():
    d = {}
    for ln in open(GOLD):
        if ln.startswith("#") or not ln.strip():
            continue
        k, *v = ln.split()
        d[k] = [float(x) for x in v]
    return d


def test_hand_worked():
    g = gold()
    cfg = oracle.RewardCfg(B=[2], beta=1.0, tau_ns=250, lat_ns=np.array([[100], [300]]),
                           arrival_ns=np.array(g["A_arrivals"], np.int64))
    r = oracle.async_serve(cfg, 2, 6, 0, acc=[0.9, 0.6])
    for k, key in (("served", "A_served"), ("overdue", "A_overdue"), ("exceed_ns", "A_exceed"),
                   ("batches", "A_batches"), ("unserved", "A_unserved")):
        assert r[k][0] == g[key][0], k
    assert r["model_batches"][0].tolist() == [int(x) for x in g["A_model_batches"]]
    assert abs(r["reward"][0] - g["A_reward"][0]) < 1e-12
    cfg = oracle.RewardCfg(B=[1, 2], beta=1.0, tau_ns=200, lat_ns=np.array([[100, 150], [50, 80]]),
                           arrival_ns=np.array(g["B_arrivals"], np.int64))
    r = oracle.async_serve(cfg, 2, 2, 0)
    for k, key in (("served", "B_served"), ("overdue", "B_overdue"), ("exceed_ns", "B_exceed"),
                   ("batches", "B_batches"), ("unserved", "B_unserved")):
        assert r[k][0] == g[key][0], k
    assert r["model_batches"][0].tolist() == [int(x) for x in g["B_model_batches"]]


def test_single_model_is_algorithm3():
    """K = 1: one server, no ensemble -- exactly the synchronous greedy policy of v = {m0}."""
    B = [16, 32, 48, 64]
    lat = lat_profile(3, B)[2:3]
    cfg = oracle.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat, rates=[128.0, 272.0, 400.0])
    a = oracle.async_serve(cfg, 1, 5000, 20_000_000)
    s = oracle.greedy_serve(cfg, 1, 5000, 20_000_000)
    for k in ("served", "overdue", "exceed_ns", "batches", "unserved"):
        np.testing.assert_array_equal(a[k], s[k][:, 0], err_msg=k)


def test_accounting():
    B = [16, 32, 48, 64]
    cfg = oracle.RewardCfg(B=B, beta=1.0, tau_ns=560_000_000, lat_ns=lat_profile(3, B), rates=[128.0, 572.0, 2000.0])
    r = oracle.async_serve(cfg, 3, 7777, 0, acc=[0.8, 0.78, 0.75])
    assert (r["served"] + r["unserved"] == 7777).all()
    assert (r["model_batches"].sum(1) == r["batches"]).all()
    assert (r["overdue"] <= r["served"]).all()
    # the asynchronous mode has more throughput than the synchronous full ensemble
    s = oracle.greedy_serve(cfg, 3, 7777, 0)
    assert (r["overdue"][1:] < s["overdue"][1:, -1]).all()
