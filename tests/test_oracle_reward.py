"""Reward / batch-moment pins for the oracle (eq. multi_acc_reward).

R1-R3: SPEC.md:627-629. R4, R5: worked by hand (tests/golden/r_reward_examples.txt).
Arrivals (reading Q9): t_s = floor(s*1e9/r) ns, global request index s.
"""
import os

import numpy as np

import oracle
from test_oracle_pins import onehot_logits

GOLD = os.path.join(os.path.dirname(__file__), "golden", "r_reward_examples.txt")


def gold():
    out = {}
    for ln in open(GOLD):
        if ln.strip() and not ln.startswith("#"):
            toks = ln.split()
            out[toks[0]] = {k: float(v) for k, v in (t.split("=") for t in toks[1:])}
    return out


def _single_model(n, n_correct):
    """K=1, C=2: n samples, the first n_correct predicted correctly (positions given)."""
    preds = np.zeros((n, 1), np.int32)
    y = np.zeros(n, np.int32)
    y[n_correct:] = 1
    return onehot_logits(preds, 2), y


def test_R1_no_overdue():
    g = gold()["R1"]
    b = int(g["b"])
    L, y = _single_model(5 * b, int(0.8 * 5 * b))  # a = 0.8 exactly
    cfg = oracle.RewardCfg(B=[b], beta=g["beta"], tau_ns=10**15, lat_ns=np.array([[1]]), rates=[1000.0])
    t = oracle.table(L, y, 1, 2, cfg=cfg)
    assert t.O[0, 0, 0] == 0
    np.testing.assert_allclose(t.reward_sur[0, 0, 0] / 5, g["reward_per_batch"], rtol=1e-15)


def test_R2_all_overdue_beta1():
    g = gold()["R2"]
    b = int(g["b"])
    L, y = _single_model(3 * b, 2 * b)
    cfg = oracle.RewardCfg(B=[b], beta=1.0, tau_ns=0, lat_ns=np.array([[1]]), rates=[1000.0])
    t = oracle.table(L, y, 1, 2, cfg=cfg)
    assert t.O[0, 0, 0] == 3 * b
    assert t.reward_sur[0, 0, 0] == g["reward_per_batch"]
    assert t.reward_lab[0, 0, 0] == 0.0


def test_R3_beta0_independent_of_overdue():
    L, y = _single_model(64, 40)
    r = []
    for tau in (0, 10**15):
        cfg = oracle.RewardCfg(B=[16, 32], beta=0.0, tau_ns=tau, lat_ns=np.array([[5, 9]]), rates=[100.0])
        r.append(oracle.table(L, y, 1, 2, cfg=cfg))
    assert (r[0].O != r[1].O).any()
    np.testing.assert_array_equal(r[0].reward_sur, r[1].reward_sur)
    np.testing.assert_array_equal(r[0].reward_lab, r[1].reward_lab)


def test_R4_uniform_arrivals_overdue_count():
    g = gold()["R4"]
    b = int(g["b"])
    nbat = 5
    L, y = _single_model(nbat * b, int(0.8 * nbat * b))
    cfg = oracle.RewardCfg(B=[b], beta=g["beta"], tau_ns=int(g["tau_ms"] * 1e6),
                           lat_ns=np.array([[int(g["c_ms"] * 1e6)]]), rates=[g["rate"]])
    t = oracle.table(L, y, 1, 2, cfg=cfg)
    assert t.O[0, 0, 0] == nbat * g["overdue_per_batch"]
    np.testing.assert_allclose(t.reward_sur[0, 0, 0] / nbat, g["reward_per_batch"], rtol=1e-14)


def test_R5_latency_equal_tau_is_not_overdue_and_exceed_time():
    g = gold()["R5"]
    b = int(g["b"])
    L, y = _single_model(2 * b + 5, 7)  # 2 complete batches + a trailing partial batch (Q13)
    cfg = oracle.RewardCfg(B=[b], beta=1.0, tau_ns=int(g["tau_ms"] * 1e6),
                           lat_ns=np.array([[int(g["c_ms"] * 1e6)]]), rates=[g["rate"]], want_exceed=True)
    t = oracle.table(L, y, 1, 2, cfg=cfg)
    assert t.O[0, 0, 0] == 2 * g["overdue_per_batch"]
    assert t.E[0, 0, 0] == 2 * g["exceed_ns_per_batch"]


def test_straggler_latency_and_labelled_moments():
    """c(v,b) = max over members; Q = sum_j corr_j * o_j."""
    K, C, b = 2, 3, 4
    # 8 samples = 2 batches; model 0 fast, model 1 slow
    preds = np.array([[0, 0], [1, 1], [2, 0], [0, 1], [0, 0], [0, 0], [1, 1], [2, 2]], np.int32)
    y = np.array([0, 1, 0, 0, 0, 1, 1, 2], np.int32)
    lat = np.array([[100], [300]])
    cfg = oracle.RewardCfg(B=[b], beta=1.0, tau_ns=250, lat_ns=lat, arrival_ns=np.arange(8) * 10, want_exceed=True)
    t = oracle.table(onehot_logits(preds, C), y, K, C, tie=oracle.TIE_LOWEST_CLASS, cfg=cfg)
    # waits in a batch: 30,20,10,0. v=1 (c=100): none overdue. v=2,3 (c=300): all 4 overdue.
    assert t.O[0, 0].tolist() == [0, 8, 8]
    assert t.E[0, 0].tolist() == [0, (80 + 70 + 60 + 50) * 2, (80 + 70 + 60 + 50) * 2]
    # per-batch vote-correct counts
    ok = np.array([[oracle.vote(preds[n], v, C, oracle.TIE_LOWEST_CLASS) == y[n] for v in (1, 2, 3)] for n in range(8)])
    corr_j = ok.reshape(2, 4, 3).sum(1)  # [batch][v]
    o_j = np.array([[0, 4, 4], [0, 4, 4]])
    assert t.corr[0].tolist() == corr_j.sum(0).tolist()
    assert t.Q[0, 0].tolist() == (corr_j * o_j).sum(0).tolist()
    np.testing.assert_allclose(t.reward_lab[0, 0], corr_j.sum(0) - (1.0 / b) * (corr_j * o_j).sum(0), rtol=1e-15)


def test_arrival_closed_form():
    assert oracle.arrival_ns(0, 128.0) == 0
    assert oracle.arrival_ns(10, 10.0) == 10**9
    assert oracle.arrival_ns(3, 572.0) == int(np.floor(3e9 / 572.0))
    # exact integer-ns comparison avoids 0.1+0.2 > 0.3 style miscounts (reading Q10)
    assert 0.2 + 0.1 > 0.3 and oracle.arrival_ns(3, 10.0) - oracle.arrival_ns(1, 10.0) == 200_000_000


def test_R6_queue_aware_worked_example():
    """Reading Q15: FIFO ensemble server, start_j = max(t_last(j), finish_{j-1})."""
    g = gold()["R6"]
    L, y = _single_model(6, 6)
    for queue, tag in ((False, "noqueue"), (True, "queue")):
        cfg = oracle.RewardCfg(B=[2], beta=1.0, tau_ns=300, lat_ns=np.array([[250]]), rates=[1e7], queue=queue)
        t = oracle.table(L, y, 1, 2, cfg=cfg)
        assert t.O[0, 0, 0] == g[f"O_{tag}"]
        assert t.E[0, 0, 0] == g[f"E_{tag}"]
        assert t.Q[0, 0, 0] == g[f"Q_{tag}"]


def test_queue_invariants():
    """Backlog only delays: O, E (queue) >= O, E (no queue) everywhere; with arrivals far apart
    (no batch ever waits) the two modes agree exactly."""
    rng = np.random.default_rng(5)
    K, C, N = 3, 5, 480
    y = rng.integers(0, C, N).astype(np.int32)
    L = rng.normal(size=(N, K, C))
    lat = np.array([[40_000_000, 70_000_000], [25_000_000, 50_000_000], [60_000_000, 90_000_000]], np.int64)
    for rates, equal in (([400.0, 1000.0], False), ([0.5], True)):
        t = {}
        for q in (False, True):
            cfg = oracle.RewardCfg(B=[16, 48], beta=1.0, tau_ns=200_000_000, lat_ns=lat, rates=rates, queue=q)
            t[q] = oracle.table(L, y, K, C, cfg=cfg)
        assert (t[True].O >= t[False].O).all() and (t[True].E >= t[False].E).all()
        if equal:
            np.testing.assert_array_equal(t[True].O, t[False].O)
            np.testing.assert_array_equal(t[True].E, t[False].E)
        else:
            assert (t[True].O > t[False].O).any()


def test_S1_greedy_batching_worked_example():
    """NEXT-1: Algorithm 3 by hand (tests/golden/r_reward_examples.txt, S1)."""
    for key in ("S1", "S1b"):
        g = gold()[key]
        cfg = oracle.RewardCfg(B=[2, 4], beta=1.0, tau_ns=1000, lat_ns=np.array([[600, 900]]), rates=[1e7])
        r = oracle.greedy_serve(cfg, 1, int(g["N"]), 50)
        for k, name in (("served", "served"), ("overdue", "overdue"), ("exceed", "exceed_ns"), ("batches", "batches"),
                        ("unserved", "unserved")):
            assert r[name][0, 0] == g[k], (key, k)


def test_greedy_batching_properties():
    """served + unserved = N; unserved < min B (after the last arrival the rule keeps dispatching
    while min B requests wait); no batch exceeds max B."""
    K, N = 3, 700
    lat = np.array([[4_000_000, 7_000_000, 9_000_000], [2_000_000, 3_000_000, 5_000_000],
                    [8_000_000, 12_000_000, 15_000_000]], np.int64)
    cfg = oracle.RewardCfg(B=[16, 32, 48], beta=1.0, tau_ns=100_000_000, lat_ns=lat, rates=[300.0, 3000.0])
    for delta in (0, 10_000_000, 100_000_000):
        r = oracle.greedy_serve(cfg, K, N, delta)
        assert ((r["served"] + r["unserved"]) == N).all()
        assert (r["unserved"] < 16).all()
        assert (r["batches"] >= r["served"] // 48).all()
