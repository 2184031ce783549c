"""Thin ctypes binding of librk.so (include/rk.h). Argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; there is no Python or CPU
compute path. If librk.so cannot be loaded the import of this module's functions raises —
there is deliberately no fallback.

Buffers may be torch tensors (``data_ptr()``), numpy arrays (host) or raw integer pointers.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

RK_OK, RK_EINVAL, RK_ESTATE, RK_ENOMEM, RK_ECUDA, RK_ENCCL, RK_ELABEL, RK_ENONFINITE, RK_EUNSUPPORTED = range(9)
TIE_BEST_MEMBER, TIE_LOWEST_CLASS = 0, 1

EXPORTS = ["rk_create", "rk_nccl_unique_id", "rk_load_ensemble", "rk_score", "rk_score_logits", "rk_subset_reset",
           "rk_subset_accumulate", "rk_subset_finalize", "rk_subset_stats", "rk_predict", "rk_greedy_serve", "rk_outputs",
           "rk_sine_arrivals", "rk_async_serve", "rk_serve_stream", "rk_ac_dims", "rk_ac_rollout", "rk_ac_grad",
           "rk_ac_apply", "rk_score_labelled", "rk_vote_diag", "rk_outputs_s2",
           "rk_group_counts",
           "rk_set_profiling", "rk_kernel_stats", "rk_last_error", "rk_status_string", "rk_destroy"]


class RkError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class _Cfg(ctypes.Structure):
    _fields_ = [("nB", ctypes.c_int), ("B", ctypes.c_void_p), ("beta", ctypes.c_double), ("tau_ns", ctypes.c_int64),
                ("lat_ns", ctypes.c_void_p), ("nR", ctypes.c_int), ("rates", ctypes.c_void_p),
                ("arrival_ns", ctypes.c_void_p), ("want_exceed", ctypes.c_int), ("want_labelled", ctypes.c_int),
                ("queue", ctypes.c_int)]


class _Table(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64)] + [(n, ctypes.c_void_p) for n in
                                          ("cnt_vote", "cnt_avg", "n_recheck", "corr", "O", "Q", "E",
                                           "reward_sur", "reward_lab")]


class _Serve(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("served", "overdue", "exceed_ns", "batches", "unserved", "reward")]


class _Sine(ctypes.Structure):
    _fields_ = [("ref_rate", ctypes.c_double), ("period_ns", ctypes.c_int64), ("delta_ns", ctypes.c_int64),
                ("noise_std", ctypes.c_double), ("seed", ctypes.c_uint64)]


class _AcCfg(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("H", ctypes.c_int), ("n_steps", ctypes.c_int), ("gamma", ctypes.c_double),
                ("reward_scale", ctypes.c_double), ("entropy", ctypes.c_double)]


class _Traj(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("states", "actions", "rewards", "overdue", "t_dec", "t_start", "t_done")]


class _KStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double),
                ("bytes", ctypes.c_double), ("flops", ctypes.c_double)]


def load_library(path: str | None = None):
    """Load (building first if stale) librk.so. Raises if it cannot be built or loaded."""
    global _lib
    if _lib is not None:
        return _lib
    so = path or os.environ.get("RK_LIB") or _build.build()  # RK_LIB: another build of librk.so (experiments)
    L = ctypes.CDLL(so)
    vp, i32, i64, u32, c = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_char_p
    L.rk_create.argtypes = [ctypes.POINTER(vp), i32, vp, i32, i32]
    L.rk_nccl_unique_id.argtypes = [vp]
    L.rk_load_ensemble.argtypes = [vp, i32, i32, i32, vp, vp, i32, vp, i32]
    L.rk_score.argtypes = [vp, vp, i64, i64, vp]
    L.rk_score_logits.argtypes = [vp, vp, i32, i64, i64, vp]
    L.rk_score_labelled.argtypes = [vp, vp, vp, i64, i64, vp]
    L.rk_vote_diag.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.rk_subset_reset.argtypes = [vp, ctypes.POINTER(_Cfg)]
    L.rk_subset_accumulate.argtypes = [vp, vp, vp]
    L.rk_subset_finalize.argtypes = [vp, ctypes.POINTER(_Table), vp]
    L.rk_subset_stats.argtypes = [vp, vp, ctypes.POINTER(_Cfg), ctypes.POINTER(_Table), vp]
    L.rk_predict.argtypes = [vp, u32, vp, vp, vp, vp]
    L.rk_greedy_serve.argtypes = [vp, ctypes.POINTER(_Cfg), i64, i64, vp, ctypes.POINTER(_Serve), vp]
    L.rk_outputs_s2.argtypes = [vp, ctypes.POINTER(vp)]
    L.rk_outputs.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(i32), ctypes.POINTER(vp), ctypes.POINTER(vp),
                             ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.rk_group_counts.argtypes = [vp, vp, i64, ctypes.POINTER(i32), ctypes.POINTER(i64), vp]
    L.rk_async_serve.argtypes = [vp, ctypes.POINTER(_Cfg), i64, i64, vp, ctypes.POINTER(_Serve), vp, vp]
    L.rk_serve_stream.argtypes = [vp, vp, i64, ctypes.POINTER(_Cfg), i64, u32, vp, vp, ctypes.POINTER(_Serve),
                                  ctypes.POINTER(i64), vp]
    L.rk_ac_dims.argtypes = [vp, i32, ctypes.POINTER(_AcCfg), ctypes.POINTER(i32), ctypes.POINTER(i32),
                             ctypes.POINTER(i64)]
    L.rk_ac_rollout.argtypes = [vp, ctypes.POINTER(_Cfg), vp, vp, i64, ctypes.POINTER(_AcCfg), vp, i32, vp, vp,
                                ctypes.c_uint64, ctypes.POINTER(_Traj), vp]
    L.rk_ac_grad.argtypes = [vp, ctypes.POINTER(_Cfg), ctypes.POINTER(_AcCfg), vp, ctypes.POINTER(_Traj), i32, vp, vp, vp]
    L.rk_ac_apply.argtypes = [vp, ctypes.POINTER(_Cfg), ctypes.POINTER(_AcCfg), vp, vp, ctypes.c_float,
                              ctypes.c_float, vp]
    L.rk_sine_arrivals.argtypes = [vp, ctypes.POINTER(_Sine), i64, i64, vp, vp]
    L.rk_set_profiling.argtypes = [vp, i32]
    L.rk_kernel_stats.argtypes = [vp, ctypes.POINTER(_KStat), i32, ctypes.POINTER(i32)]
    for f in EXPORTS:
        if f not in ("rk_last_error", "rk_status_string", "rk_destroy"):
            getattr(L, f).restype = i32
    L.rk_last_error.argtypes = [vp]
    L.rk_last_error.restype = c
    L.rk_status_string.argtypes = [i32]
    L.rk_status_string.restype = c
    L.rk_destroy.argtypes = [vp]
    L.rk_destroy.restype = None
    _lib = L
    return L


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)}")


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = L.rk_nccl_unique_id(buf)
    if rc != RK_OK:
        raise RkError(rc, "rk_nccl_unique_id failed")
    return buf.raw


@dataclass
class RewardCfg:
    """rk_reward_cfg. lat_ns is [K][nB] int64; rates in req/s (or arrival_ns per chunk)."""
    B: list
    beta: float
    tau_ns: int
    lat_ns: np.ndarray
    rates: list | None = None
    arrival_ns: object = None
    want_exceed: bool = True
    want_labelled: bool = True
    queue: bool = False  # reading Q15: FIFO ensemble server, batch j waits for batch j-1


class Context:
    """One rk_ctx (one GPU rank)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self._L = load_library()
        self._p = ctypes.c_void_p()
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(nccl_id, 128)
        rc = self._L.rk_create(ctypes.byref(self._p), device, idbuf, rank, world)
        if rc != RK_OK:
            raise RkError(rc, f"rk_create(device={device}, rank={rank}, world={world}) failed")
        self.K = self.C = self.S = 0
        self.cfg = None
        self._keep = []

    def _chk(self, rc, what):
        if rc != RK_OK:
            msg = self._L.rk_last_error(self._p).decode()
            raise RkError(rc, f"{what}: {msg}")

    def close(self):
        if self._p:
            self._L.rk_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- A1 setup --
    def load_ensemble(self, K, C, D=0, W=None, bias=None, scale_log2=0, member_rank=None, tie=TIE_BEST_MEMBER):
        r = None if member_rank is None else np.ascontiguousarray(member_rank, dtype=np.int32)
        self._chk(self._L.rk_load_ensemble(self._p, K, C, D, _ptr(W), _ptr(bias), scale_log2, _ptr(r), tie),
                  "rk_load_ensemble")
        self.K, self.C, self.S = K, C, (1 << K) - 1

    def score(self, X, N, offset=0, stream=None):
        self._chk(self._L.rk_score(self._p, _ptr(X), N, offset, _stream(stream)), "rk_score")

    def score_labelled(self, X, labels, N, offset=0, stream=None):
        """NEXT-3: fused forward + vote (labels known at scoring time; no logits stored for K <= 8, C > 128)."""
        self._chk(self._L.rk_score_labelled(self._p, _ptr(X), _ptr(labels), N, offset, _stream(stream)),
                  "rk_score_labelled")

    def score_logits(self, logits, ldc, N, offset=0, stream=None):
        self._chk(self._L.rk_score_logits(self._p, _ptr(logits), ldc, N, offset, _stream(stream)), "rk_score_logits")

    # -- A2-A7 --
    def _cfg(self, cfg: RewardCfg | None):
        if cfg is None:
            return None
        B = np.ascontiguousarray(cfg.B, dtype=np.int32)
        lat = np.ascontiguousarray(cfg.lat_ns, dtype=np.int64).reshape(-1)
        rates = None if cfg.rates is None else np.ascontiguousarray(cfg.rates, dtype=np.float64)
        arr = cfg.arrival_ns
        if isinstance(arr, np.ndarray):
            arr = np.ascontiguousarray(arr, dtype=np.int64)
        nR = 1 if arr is not None else (0 if rates is None else rates.size)
        self._keep = [B, lat, rates, arr]
        return _Cfg(B.size, _ptr(B), cfg.beta, int(cfg.tau_ns), _ptr(lat), nR, _ptr(rates), _ptr(arr),
                    int(cfg.want_exceed), int(cfg.want_labelled), int(cfg.queue))

    def subset_reset(self, cfg: RewardCfg | None = None):
        c = self._cfg(cfg)
        self.cfg = cfg
        self._chk(self._L.rk_subset_reset(self._p, ctypes.byref(c) if c is not None else None), "rk_subset_reset")

    def subset_accumulate(self, labels, stream=None):
        self._chk(self._L.rk_subset_accumulate(self._p, _ptr(labels), _stream(stream)), "rk_subset_accumulate")

    def _alloc_table(self):
        S = self.S
        cfg = self.cfg
        nB = len(cfg.B) if cfg is not None else 0
        nR = (1 if cfg.arrival_ns is not None else len(cfg.rates or [])) if cfg is not None else 0
        if nB == 0:
            nR = 0
        t = {"cnt_vote": np.zeros(S, np.uint64), "cnt_avg": np.zeros(S, np.uint64), "n_recheck": np.zeros(S, np.uint64),
             "corr": np.zeros((nB, S), np.uint64), "O": np.zeros((nR, nB, S), np.uint64),
             "Q": np.zeros((nR, nB, S), np.uint64), "E": np.zeros((nR, nB, S), np.uint64),
             "reward_sur": np.zeros((nR, nB, S), np.float64), "reward_lab": np.zeros((nR, nB, S), np.float64)}
        ct = _Table(0, *[_ptr(t[k]) for k in ("cnt_vote", "cnt_avg", "n_recheck", "corr", "O", "Q", "E",
                                              "reward_sur", "reward_lab")])
        return t, ct

    def subset_finalize(self, stream=None) -> dict:
        t, ct = self._alloc_table()
        self._chk(self._L.rk_subset_finalize(self._p, ctypes.byref(ct), _stream(stream)), "rk_subset_finalize")
        t["N"] = ct.N
        return t

    def subset_stats(self, labels, cfg: RewardCfg | None = None, stream=None) -> dict:
        c = self._cfg(cfg)
        self.cfg = cfg
        t, ct = self._alloc_table()
        self._chk(self._L.rk_subset_stats(self._p, _ptr(labels), ctypes.byref(c) if c is not None else None,
                                          ctypes.byref(ct), _stream(stream)), "rk_subset_stats")
        t["N"] = ct.N
        return t

    def predict(self, v, pred_vote=None, pred_avg=None, avgprob=None, stream=None):
        self._chk(self._L.rk_predict(self._p, v, _ptr(pred_vote), _ptr(pred_avg), _ptr(avgprob), _stream(stream)),
                  "rk_predict")

    def greedy_serve(self, cfg: RewardCfg, N: int, delta_ns: int, acc=None, stream=None) -> dict:
        """NEXT-1: Algorithm 3 greedy batching of every subset, per rate: arrays
        [nR][S] of served, overdue, exceed_ns, batches, unserved and (with acc [S]) reward."""
        c = self._cfg(cfg)
        nR = c.nR
        res = {k: np.zeros((nR, self.S), np.uint64) for k in ("served", "overdue", "exceed_ns", "batches", "unserved")}
        res["reward"] = np.zeros((nR, self.S), np.float64)
        a = None if acc is None else np.ascontiguousarray(acc, dtype=np.float64)
        o = _Serve(*[res[k].ctypes.data for k in ("served", "overdue", "exceed_ns", "batches", "unserved", "reward")])
        self._chk(self._L.rk_greedy_serve(self._p, ctypes.byref(c), N, delta_ns, _ptr(a), ctypes.byref(o),
                                          _stream(stream)), "rk_greedy_serve")
        if a is None:
            del res["reward"]
        return res

    def async_serve(self, cfg: RewardCfg, N: int, delta_ns: int, acc=None, stream=None) -> dict:
        """NEXT-1 baseline: all models asynchronously, one model per batch (reading S2): arrays
        [nR] of served, overdue, exceed_ns, batches, unserved, (with acc [K]) reward, and model_batches [nR][K]."""
        c = self._cfg(cfg)
        nR = c.nR
        res = {k: np.zeros(nR, np.uint64) for k in ("served", "overdue", "exceed_ns", "batches", "unserved")}
        res["reward"] = np.zeros(nR, np.float64)
        res["model_batches"] = np.zeros((nR, self.K), np.uint64)
        a = None if acc is None else np.ascontiguousarray(acc, dtype=np.float64)
        o = _Serve(*[res[k].ctypes.data for k in ("served", "overdue", "exceed_ns", "batches", "unserved", "reward")])
        self._chk(self._L.rk_async_serve(self._p, ctypes.byref(c), N, delta_ns, _ptr(a), ctypes.byref(o),
                                         res["model_batches"].ctypes.data, _stream(stream)), "rk_async_serve")
        if a is None:
            del res["reward"]
        return res

    def serve_stream(self, X, N, cfg: RewardCfg, delta_ns, v, pred_vote=None, pred_avg=None, stream=None) -> dict:
        """NEXT-1 serving loop: Algorithm 3 batches of action v, each run through the heads and the prediction
        of v; per-request predictions into the device buffers (-1 = unserved). Returns the counters."""
        c = self._cfg(cfg)
        res = {k: np.zeros(1, np.uint64) for k in ("served", "overdue", "exceed_ns", "batches", "unserved")}
        o = _Serve(*[res[k].ctypes.data for k in ("served", "overdue", "exceed_ns", "batches", "unserved")], None)
        nb = ctypes.c_int64()
        self._chk(self._L.rk_serve_stream(self._p, _ptr(X), N, ctypes.byref(c), delta_ns, v, _ptr(pred_vote),
                                          _ptr(pred_avg), ctypes.byref(o), ctypes.byref(nb), _stream(stream)),
                  "rk_serve_stream")
        return {k: int(res[k][0]) for k in res}

    # -- NEXT-2: actor-critic scheduler (argument marshalling; the loop lives in scheduler.py) --
    @staticmethod
    def _ac(ac):
        return _AcCfg(int(ac["L"]), int(ac["H"]), int(ac["n_steps"]), float(ac["gamma"]), float(ac["reward_scale"]),
                      float(ac.get("entropy", 0.0)))

    def ac_dims(self, nB, ac):
        F, A, P = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        self._chk(self._L.rk_ac_dims(self._p, nB, ctypes.byref(self._ac(ac)), ctypes.byref(F), ctypes.byref(A),
                                     ctypes.byref(P)), "rk_ac_dims")
        return F.value, A.value, P.value

    @staticmethod
    def _traj(tr):
        return _Traj(*[_ptr(tr.get(k)) for k in ("states", "actions", "rewards", "overdue", "t_dec", "t_start",
                                                  "t_done")])

    def ac_rollout(self, cfg: RewardCfg, acc, arrival, Narr, ac, params, E, h0, traj: dict, forced=None, seed=0,
                   stream=None):
        c = self._cfg(cfg)
        a = np.ascontiguousarray(acc, dtype=np.float64)
        t = self._traj(traj)
        self._chk(self._L.rk_ac_rollout(self._p, ctypes.byref(c), _ptr(a), _ptr(arrival), int(Narr),
                                        ctypes.byref(self._ac(ac)), _ptr(params), int(E), _ptr(h0), _ptr(forced),
                                        int(seed), ctypes.byref(t), _stream(stream)), "rk_ac_rollout")

    def ac_grad(self, cfg: RewardCfg, ac, params, traj: dict, E, grad, stream=None):
        c = self._cfg(cfg)
        t = self._traj(traj)
        losses = np.zeros(2, np.float64)
        self._chk(self._L.rk_ac_grad(self._p, ctypes.byref(c), ctypes.byref(self._ac(ac)), _ptr(params),
                                     ctypes.byref(t), int(E), _ptr(grad), losses.ctypes.data, _stream(stream)),
                  "rk_ac_grad")
        return losses

    def ac_apply(self, cfg: RewardCfg, ac, params, grad, lr_pi, lr_v, stream=None):
        c = self._cfg(cfg)
        self._chk(self._L.rk_ac_apply(self._p, ctypes.byref(c), ctypes.byref(self._ac(ac)), _ptr(params), _ptr(grad),
                                      float(lr_pi), float(lr_v), _stream(stream)), "rk_ac_apply")

    def sine_arrivals(self, out, N, ref_rate, period_ns, delta_ns, noise_std=0.1, seed=0, n0=0, stream=None):
        """NEXT-4: arrival times (int64 ns) of global requests [n0, n0 + N) of the sine-plus-noise process
        (reading Q16) into the device buffer `out` [N]."""
        c = _Sine(float(ref_rate), int(period_ns), int(delta_ns), float(noise_std), int(seed))
        self._chk(self._L.rk_sine_arrivals(self._p, ctypes.byref(c), int(n0), int(N), _ptr(out), _stream(stream)),
                  "rk_sine_arrivals")

    def outputs(self):
        lg, t1, mx, ls = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        ldc, n = ctypes.c_int(), ctypes.c_int64()
        self._chk(self._L.rk_outputs(self._p, ctypes.byref(lg), ctypes.byref(ldc), ctypes.byref(t1), ctypes.byref(mx),
                                     ctypes.byref(ls), ctypes.byref(n)), "rk_outputs")
        return {"logits": lg.value, "ldc": ldc.value, "top1": t1.value, "rmax": mx.value, "lsum": ls.value,
                "N": n.value}

    def outputs_s2(self):
        """Device pointer of the last rk_score batch's second-largest logits [N][K] fp32, or None."""
        s2 = ctypes.c_void_p()
        self._chk(self._L.rk_outputs_s2(self._p, ctypes.byref(s2)), "rk_outputs_s2")
        return s2.value

    def group_counts(self, stream=None):
        """Per-(group, subset) vote-correct counts of the last accumulated chunk: (gs, uint8 [groups][S])."""
        gs, ng = ctypes.c_int(), ctypes.c_int64()
        self._chk(self._L.rk_group_counts(self._p, None, 0, ctypes.byref(gs), ctypes.byref(ng), _stream(stream)),
                  "rk_group_counts")
        out = np.zeros((ng.value, self.S), np.uint8)
        if out.size:
            self._chk(self._L.rk_group_counts(self._p, out.ctypes.data, out.size, None, None, _stream(stream)),
                      "rk_group_counts")
        return gs.value, out

    def vote_diag(self):
        """(worklist, fallback, rows_skipped) counts of the last accumulated chunk (K <= 8 path)."""
        w, f, k = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._chk(self._L.rk_vote_diag(self._p, ctypes.byref(w), ctypes.byref(f), ctypes.byref(k)), "rk_vote_diag")
        return w.value, f.value, k.value

    def set_profiling(self, on: bool):
        self._chk(self._L.rk_set_profiling(self._p, int(on)), "rk_set_profiling")

    def kernel_stats(self) -> dict:
        arr = (_KStat * 16)()
        n = ctypes.c_int()
        self._chk(self._L.rk_kernel_stats(self._p, arr, 16, ctypes.byref(n)), "rk_kernel_stats")
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].total_ms, "bytes": arr[i].bytes,
                                       "flops": arr[i].flops} for i in range(min(n.value, 16))}


def action_index(v: int, b_index: int, nB: int) -> int:
    """RL action index of (subset v, batch size B[b_index]) (SPEC.md:603-611 ordering)."""
    if v <= 0:
        raise ValueError("v = 0 is excluded from the action space (PAPER.md:429)")
    return (v - 1) * nB + b_index


def action_decode(index: int, K: int, nB: int):
    n = ((1 << K) - 1) * nB
    if not 0 <= index < n:
        raise ValueError("action index out of range")
    return index // nB + 1, index % nB
