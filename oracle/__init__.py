"""CPU oracle for the Rafiki ensemble-subset hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product path
(``paper_1804_06087_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``oracle.c`` (plain C, fp64/int64). Functions follow PAPER.md
definitions (see oracle.h for citations). Every function here is pinned by
``tests/test_oracle_*.py`` against hand-computed examples, closed forms, invariants and
an independently written brute-force formulation.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

TIE_BEST_MEMBER = 0
TIE_LOWEST_CLASS = 1
OK, EINVAL, ELABEL, ENONFINITE = 0, 1, 6, 7


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle.h")]
    stale = not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in srcs)
    if force or stale:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, srcs[0], "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Cfg(ctypes.Structure):
    _fields_ = [("nB", ctypes.c_int), ("B", ctypes.c_void_p), ("beta", ctypes.c_double),
                ("tau_ns", ctypes.c_int64), ("lat_ns", ctypes.c_void_p), ("nR", ctypes.c_int),
                ("rates", ctypes.c_void_p), ("arrival_ns", ctypes.c_void_p), ("want_exceed", ctypes.c_int),
                ("queue", ctypes.c_int)]


class _Table(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("cnt_vote", "cnt_avg", "n_amb", "corr", "O", "Q", "E", "reward_sur", "reward_lab", "vote_ok",
                 "avg_ok")]


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i32, i64, u32, vp, dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double
        L.or_top1_f32.argtypes = [vp, i32]; L.or_top1_f32.restype = i32
        L.or_top1_f64.argtypes = [vp, i32]; L.or_top1_f64.restype = i32
        L.or_softmax.argtypes = [vp, i32, vp]; L.or_softmax.restype = None
        L.or_lse.argtypes = [vp, i32]; L.or_lse.restype = dbl
        L.or_vote.argtypes = [vp, i32, i32, u32, vp, i32]; L.or_vote.restype = i32
        L.or_avg.argtypes = [vp, i32, i32, u32, vp, vp]; L.or_avg.restype = i32
        L.or_logits_gemm.argtypes = [vp, vp, vp, i64, i32, i32, i32, i32, vp, i32]; L.or_logits_gemm.restype = None
        L.or_table_build.argtypes = [vp, i32, vp, i64, i32, i32, vp, vp, i32, ctypes.POINTER(_Cfg),
                                     ctypes.POINTER(_Table), i32]
        L.or_table_build.restype = i32
        L.or_predict.argtypes = [vp, i32, vp, i64, i32, i32, u32, vp, i32, vp, vp, vp, vp, vp, i32]
        L.or_predict.restype = i32
        L.or_arrival_ns.argtypes = [i64, dbl]; L.or_arrival_ns.restype = i64
        L.or_sine_params.argtypes = [dbl, vp, vp]; L.or_sine_params.restype = None
        L.or_sine_count.argtypes = [dbl, i64, i64, dbl, ctypes.c_uint64, i64]; L.or_sine_count.restype = i64
        L.or_sine_arrivals.argtypes = [dbl, i64, i64, dbl, ctypes.c_uint64, i64, i64, vp]
        L.or_sine_arrivals.restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _threads():
    return max(1, os.cpu_count() or 1)


# ---- elementary definitions ----------------------------------------------------------------
def top1(row) -> int:
    r = np.ascontiguousarray(row)
    if r.dtype == np.float32:
        return lib().or_top1_f32(_p(r), r.size)
    r = np.ascontiguousarray(r, dtype=np.float64)
    return lib().or_top1_f64(_p(r), r.size)


def softmax(l) -> np.ndarray:
    l = np.ascontiguousarray(l, dtype=np.float64)
    p = np.empty_like(l)
    lib().or_softmax(_p(l), l.size, _p(p))
    return p


def lse(l) -> float:
    l = np.ascontiguousarray(l, dtype=np.float64)
    return lib().or_lse(_p(l), l.size)


def vote(top1s, v: int, C: int, tie: int = TIE_BEST_MEMBER, rank=None) -> int:
    t = np.ascontiguousarray(top1s, dtype=np.int32)
    r = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
    return lib().or_vote(_p(t), t.size, C, v, _p(r), tie)


def avg(p, v: int):
    """p: [K][C] fp64 probabilities. Returns (pred, ambiguous, avg_vector)."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    K, C = p.shape
    amb = ctypes.c_int(0)
    out = np.empty(C, dtype=np.float64)
    pred = lib().or_avg(_p(p), K, C, v, ctypes.byref(amb), _p(out))
    return pred, bool(amb.value), out


def arrival_ns(s: int, rate: float) -> int:
    return lib().or_arrival_ns(s, rate)


def sine_params(ref: float):
    """(k, b) of rate(t) = k sin(2 pi t / T) + b (eqs. eq:r1/eq:r2, reading Q16)."""
    k, b = ctypes.c_double(), ctypes.c_double()
    lib().or_sine_params(ref, ctypes.byref(k), ctypes.byref(b))
    return k.value, b.value


def sine_count(ref: float, period_ns: int, delta_ns: int, sigma: float, seed: int, j: int) -> int:
    """Requests added by simulator invocation j (reading Q16)."""
    return lib().or_sine_count(ref, period_ns, delta_ns, sigma, seed, j)


def sine_arrivals(ref: float, period_ns: int, delta_ns: int, sigma: float, seed: int, n0: int, N: int) -> np.ndarray:
    """Arrival times (ns) of global requests [n0, n0 + N) of the sine-plus-noise process (reading Q16)."""
    out = np.zeros(N, np.int64)
    rc = lib().or_sine_arrivals(ref, period_ns, delta_ns, sigma, seed, n0, N, _p(out))
    if rc != OK:
        raise ValueError(f"or_sine_arrivals failed ({rc})")
    return out


def logits_gemm(X_bits, W_bits, bias, scale_log2: int) -> np.ndarray:
    """fp64 logits [N][K][C] of the synthetic dense heads (step A1)."""
    X = np.ascontiguousarray(X_bits, dtype=np.uint16)
    W = np.ascontiguousarray(W_bits, dtype=np.uint16)
    N, D = X.shape
    K, C, D2 = W.shape
    assert D == D2
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    out = np.empty((N, K, C), dtype=np.float64)
    lib().or_logits_gemm(_p(X), _p(W), _p(b), N, K, C, D, scale_log2, _p(out), _threads())
    return out


# ---- table -------------------------------------------------------------------------------------
@dataclass
class RewardCfg:
    B: list
    beta: float
    tau_ns: int
    lat_ns: np.ndarray          # [K][nB] int64
    rates: list | None = None   # req/s
    arrival_ns: np.ndarray | None = None
    want_exceed: bool = True
    queue: bool = False         # reading Q15: FIFO ensemble server, batch j waits for batch j-1


@dataclass
class Table:
    cnt_vote: np.ndarray
    cnt_avg: np.ndarray
    n_amb: np.ndarray
    corr: np.ndarray | None = None
    O: np.ndarray | None = None
    Q: np.ndarray | None = None
    E: np.ndarray | None = None
    reward_sur: np.ndarray | None = None
    reward_lab: np.ndarray | None = None
    vote_ok: np.ndarray | None = None   # [N][S] uint8 per-sample vote correctness (want_bits)
    avg_ok: np.ndarray | None = None    # [N][S] uint8 per-sample average correctness (want_bits)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


def table(logits, labels, K: int, C: int, tie: int = TIE_BEST_MEMBER, rank=None,
          cfg: RewardCfg | None = None, threads: int | None = None, want_bits: bool = False) -> Table:
    """Steps A2-A7 over the whole dataset. logits: fp32 [N][K][ldc] or fp64 [N][K][C].
    want_bits: also return the per-sample correctness bits vote_ok / avg_ok [N][S] (uint8)."""
    lg = np.ascontiguousarray(logits)
    N = lg.shape[0]
    lf = ld = None
    ldc = 0
    if lg.dtype == np.float32:
        lf, ldc = lg, lg.shape[2]
    else:
        ld = np.ascontiguousarray(lg, dtype=np.float64)
        assert ld.shape[2] == C
    y = np.ascontiguousarray(labels, dtype=np.int32)
    assert y.shape[0] == N
    r = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
    S = (1 << K) - 1
    keep = []
    cc = None
    nB = nR = 0
    if cfg is not None:
        nB = len(cfg.B)
        Bv = np.ascontiguousarray(cfg.B, dtype=np.int32)
        lat = np.ascontiguousarray(cfg.lat_ns, dtype=np.int64).reshape(K, nB)
        if cfg.arrival_ns is not None:
            arr = np.ascontiguousarray(cfg.arrival_ns, dtype=np.int64)
            rates = None
            nR = 1
        else:
            arr = None
            rates = np.ascontiguousarray(cfg.rates, dtype=np.float64)
            nR = rates.size
        keep += [Bv, lat, arr, rates]
        cc = _Cfg(nB, _p(Bv), cfg.beta, cfg.tau_ns, _p(lat), nR, _p(rates), _p(arr), int(cfg.want_exceed),
                  int(cfg.queue))
    t = Table(np.zeros(S, np.uint64), np.zeros(S, np.uint64), np.zeros(S, np.uint64))
    if cfg is not None:
        t.corr = np.zeros((nB, S), np.uint64)
        t.O = np.zeros((nR, nB, S), np.uint64)
        t.Q = np.zeros((nR, nB, S), np.uint64)
        t.E = np.zeros((nR, nB, S), np.uint64) if cfg.want_exceed else None
        t.reward_sur = np.zeros((nR, nB, S), np.float64)
        t.reward_lab = np.zeros((nR, nB, S), np.float64)
    if want_bits:
        t.vote_ok = np.zeros((N, S), np.uint8)
        t.avg_ok = np.zeros((N, S), np.uint8)
    ct = _Table(_p(t.cnt_vote), _p(t.cnt_avg), _p(t.n_amb), _p(t.corr), _p(t.O), _p(t.Q), _p(t.E),
                _p(t.reward_sur), _p(t.reward_lab), _p(t.vote_ok), _p(t.avg_ok))
    rc = lib().or_table_build(_p(lf), ldc, _p(ld), N, K, C, _p(y), _p(r), tie,
                              ctypes.byref(cc) if cc is not None else None, ctypes.byref(ct),
                              threads or _threads())
    if rc != OK:
        raise OracleError(rc)
    return t


def predict(logits, K: int, C: int, v: int, tie: int = TIE_BEST_MEMBER, rank=None, want_avgprob=False):
    """Per-sample (pred_vote, pred_avg, avgprob|None, top1 [N][K], lse [N][K]) for action v."""
    lg = np.ascontiguousarray(logits)
    N = lg.shape[0]
    lf = ld = None
    ldc = 0
    if lg.dtype == np.float32:
        lf, ldc = lg, lg.shape[2]
    else:
        ld = np.ascontiguousarray(lg, dtype=np.float64)
    r = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
    pv = np.empty(N, np.int32)
    pa = np.empty(N, np.int32)
    ap = np.empty((N, C), np.float64) if want_avgprob else None
    t1 = np.empty((N, K), np.int32)
    ls = np.empty((N, K), np.float64)
    rc = lib().or_predict(_p(lf), ldc, _p(ld), N, K, C, v, _p(r), tie, _p(pv), _p(pa), _p(ap), _p(t1), _p(ls), 1)
    if rc != OK:
        raise OracleError(rc)
    return pv, pa, ap, t1, ls


# ---- NEXT-1: Algorithm 3 greedy batching ------------------------------------------------------
class _Serve(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("served", "overdue", "exceed_ns", "batches", "unserved")]


def greedy_serve(cfg: RewardCfg, K: int, N: int, delta_ns: int) -> dict:
    """Algorithm 3 per (rate, subset): arrays [nR][S] of served, overdue,
    exceed_ns, batches, unserved (reading S1)."""
    nB = len(cfg.B)
    Bv = np.ascontiguousarray(cfg.B, dtype=np.int32)
    lat = np.ascontiguousarray(cfg.lat_ns, dtype=np.int64).reshape(K, nB)
    if cfg.arrival_ns is not None:
        arr, rates, nR = np.ascontiguousarray(cfg.arrival_ns, dtype=np.int64), None, 1
    else:
        arr, rates = None, np.ascontiguousarray(cfg.rates, dtype=np.float64)
        nR = rates.size
    cc = _Cfg(nB, _p(Bv), cfg.beta, cfg.tau_ns, _p(lat), nR, _p(rates), _p(arr), int(cfg.want_exceed),
              int(cfg.queue))
    S = (1 << K) - 1
    out = (_Serve * (nR * S))()
    L = lib()
    L.or_greedy_serve.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
    rc = L.or_greedy_serve(ctypes.byref(cc), K, N, delta_ns, out)
    if rc != OK:
        raise OracleError(rc)
    res = {}
    for name in ("served", "overdue", "exceed_ns", "batches", "unserved"):
        res[name] = np.array([getattr(o, name) for o in out], dtype=np.uint64).reshape(nR, S)
    return res


def async_serve(cfg: RewardCfg, K: int, N: int, delta_ns: int, acc=None) -> dict:
    """The asynchronous one-model-per-batch baseline (reading S2), per rate: arrays
    [nR] of served, overdue, exceed_ns, batches, unserved, reward (with acc [K]) and batches per model [nR][K]."""
    nB = len(cfg.B)
    Bv = np.ascontiguousarray(cfg.B, dtype=np.int32)
    lat = np.ascontiguousarray(cfg.lat_ns, dtype=np.int64).reshape(K, nB)
    if cfg.arrival_ns is not None:
        arr, rates, nR = np.ascontiguousarray(cfg.arrival_ns, dtype=np.int64), None, 1
    else:
        arr, rates = None, np.ascontiguousarray(cfg.rates, dtype=np.float64)
        nR = rates.size
    cc = _Cfg(nB, _p(Bv), cfg.beta, cfg.tau_ns, _p(lat), nR, _p(rates), _p(arr), int(cfg.want_exceed), 0)
    out = (_Serve * nR)()
    rew = np.zeros(nR, np.float64)
    mb = np.zeros((nR, K), np.uint64)
    a = None if acc is None else np.ascontiguousarray(acc, dtype=np.float64)
    L = lib()
    L.or_async_serve.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    rc = L.or_async_serve(ctypes.byref(cc), K, N, delta_ns, _p(a), out, _p(rew), _p(mb))
    if rc != OK:
        raise OracleError(rc)
    res = {name: np.array([getattr(o, name) for o in out], dtype=np.uint64)
           for name in ("served", "overdue", "exceed_ns", "batches", "unserved")}
    res["model_batches"] = mb
    if a is not None:
        res["reward"] = rew
    return res


# ---- NEXT-2: RL environment and actor-critic gradients (reading S3) -------------------------------
class _Env(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("nB", ctypes.c_int), ("L", ctypes.c_int), ("B", ctypes.c_void_p),
                ("lat_ns", ctypes.c_void_p), ("tau_ns", ctypes.c_int64), ("beta", ctypes.c_double),
                ("acc", ctypes.c_void_p), ("arrival", ctypes.c_void_p), ("Narr", ctypes.c_int64)]


def env_rollout(K: int, B, lat_ns, tau_ns: int, beta: float, acc, arrival, L: int, actions, h0: int) -> dict:
    """One episode of the scheduler's environment under the given actions (reading S3):
    states [n][F], rewards, overdue, t_dec, t_start, t_done."""
    Bv = np.ascontiguousarray(B, dtype=np.int32)
    lat = np.ascontiguousarray(lat_ns, dtype=np.int64).reshape(K, len(B))
    a = np.ascontiguousarray(acc, dtype=np.float64)
    arr = np.ascontiguousarray(arrival, dtype=np.int64)
    act = np.ascontiguousarray(actions, dtype=np.int32)
    n = act.size
    F = L + K * len(B) + K
    env = _Env(K, len(B), L, _p(Bv), _p(lat), int(tau_ns), float(beta), _p(a), _p(arr), arr.size)
    out = {"states": np.zeros((n, F), np.float32), "rewards": np.zeros(n), "overdue": np.zeros(n, np.int32),
           "t_dec": np.zeros(n, np.int64), "t_start": np.zeros(n, np.int64), "t_done": np.zeros(n, np.int64)}
    L_ = lib()
    L_.or_env_rollout.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 6
    rc = L_.or_env_rollout(ctypes.byref(env), _p(act), n, h0, *[_p(out[k]) for k in
                                                                 ("states", "rewards", "overdue", "t_dec", "t_start",
                                                                  "t_done")])
    if rc != OK:
        raise OracleError(rc)
    return out


def ac_param_count(F: int, H: int, A: int) -> int:
    return H * F + H + A * H + A + H * F + H + H + 1


def ac_grad(F: int, H: int, A: int, params, states, actions, rewards, gamma: float, scale: float, ent: float = 0.0):
    """Actor-critic gradients in fp64 (PAPER.md:123-131 eqs. eq:dJ / eq:hatJ with the baseline V(s_t)):
    (grad [flat], loss_pi, loss_v) for E episodes x n steps (states [E][n][F], actions/rewards [E][n])."""
    P = np.ascontiguousarray(params, dtype=np.float64)
    st = np.ascontiguousarray(states, dtype=np.float32)
    act = np.ascontiguousarray(actions, dtype=np.int32)
    rew = np.ascontiguousarray(rewards, dtype=np.float64)
    E, n = act.shape
    g = np.zeros(ac_param_count(F, H, A), np.float64)
    lp, lv = ctypes.c_double(), ctypes.c_double()
    L_ = lib()
    L_.or_ac_grad.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                                          ctypes.c_double, ctypes.c_double,
                                                                          ctypes.c_void_p, ctypes.c_void_p,
                                                                          ctypes.c_void_p]
    rc = L_.or_ac_grad(F, H, A, _p(P), _p(st), _p(act), _p(rew), E, n, gamma, scale, ent, _p(g), ctypes.byref(lp),
                       ctypes.byref(lv))
    if rc != OK:
        raise OracleError(rc)
    return g, lp.value, lv.value
