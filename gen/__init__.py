"""Seeded synthetic input generators (shared by the oracle side and the GPU side).

Holds no arithmetic of the method (see rk_gen.h). Host fills return numpy arrays; device
fills write into caller-owned device memory (raw pointers, e.g. ``tensor.data_ptr()``).

The workload recipe ("Input recipe"):
  * labels uniform in [0, C);
  * logits by the SURVEY.md §8(d) correlated formula (dyadic, Irwin-Hall noise);
  * GEMM features X [N][D] / head weights W [K][C][D] in bf16: prototype-matched heads.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_HERE, "libgen_host.so")
_DEV_SO = os.path.join(_HERE, "libgen_cuda.so")
_host = None
_dev = None

# Calibrated parameters (tests/test_gen.py checks the bands).
Q24 = 1 << 24


def logit_params(K: int, C: int):
    """(mu0_q24, dmu_q24) for the logits formula. Dyadic values only."""
    if C <= 10:
        mu0, dmu = 2.5, 0.125
    elif C <= 100:
        mu0, dmu = 3.125, 0.03125
    else:
        mu0, dmu = 4.0, 0.0625 if K <= 6 else 0.046875
    return int(mu0 * Q24), int(dmu * Q24)


# GEMM heads: psig (fraction of prototype-matched feature dims) and flip rates, all /65536.
def head_params(D: int, C: int, K: int):
    """(psig_q16, flip0_q16, dflip_q16, scale_log2) for the dense heads. Logit = 2^scale_log2 * x.w."""
    # C = 1000 calibrated to SURVEY.md §8(d)'s Inception-like bands (scripts/calibrate_heads.py, DESIGN.md
    # §4): K = 8 per-model top-1 0.82..0.76, 56% unanimous, mean max-softmax 0.77, mean |S_c| 7.4, full-set
    # average gain +4.4 points; psig packs P(matched dim) = 4250/65536 and P(noise dim != 0) = 25600/65536
    # (rk_gen.h rkg_x_int). C = 100 (c5, D = 1024) calibrated to §8(d)'s K = 12 row: per-model top-1 0.78..0.77,
    # 50 % unanimous, mean max-softmax 0.79, |S_c| 6.8, full-set average 0.84 (round 1: 5800/800/80 gave 35 %).
    if C <= 10:
        return 3800, 800, 150, -3
    if C <= 100:
        return 6200, 50, 80, -3
    return 4250 | (25600 << 16), 50, 250, -3


def _src(*names):
    return [os.path.join(_HERE, n) for n in names]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_host(force: bool = False) -> str:
    srcs = _src("gen_host.c", "rk_gen.h")
    if force or _stale(_HOST_SO, srcs):
        tmp = _HOST_SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", tmp,
                               _src("gen_host.c")[0], "-lm"])
        os.replace(tmp, _HOST_SO)
    return _HOST_SO


def build_device(force: bool = False) -> str:
    srcs = _src("gen_cuda.cu", "rk_gen.h")
    if force or _stale(_DEV_SO, srcs):
        tmp = _DEV_SO + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _src("gen_cuda.cu")[0]])
        os.replace(tmp, _DEV_SO)
    return _DEV_SO


def _lib():
    global _host
    if _host is None:
        L = ctypes.CDLL(build_host())
        i64, u64, i32, u32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
        L.rkg_fill_labels.argtypes = [u64, i64, i64, i32, vp, i32]
        L.rkg_fill_logits.argtypes = [u64, i64, i64, i32, i32, i32, i64, i64, vp, vp, i32]
        L.rkg_fill_x.argtypes = [u64, i64, i64, i32, i32, u32, i32, vp, vp, i32]
        L.rkg_fill_w.argtypes = [u64, i32, i32, i32, u32, u32, i32, vp, i32]
        L.rkg_fill_bias.argtypes = [u64, i32, i32, i32, vp]
        for f in (L.rkg_fill_labels, L.rkg_fill_logits, L.rkg_fill_x, L.rkg_fill_w, L.rkg_fill_bias):
            f.restype = None
        _host = L
    return _host


def _threads():
    return max(1, os.cpu_count() or 1)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def labels(seed: int, n0: int, n: int, C: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    _lib().rkg_fill_labels(seed, n0, n, C, _p(out), _threads())
    return out


def logits(seed: int, n0: int, n: int, K: int, C: int, ldc: int | None = None, params=None,
           y: np.ndarray | None = None) -> np.ndarray:
    """fp32 logits [n][K][ldc]; columns >= C are NaN (never read by the method)."""
    ldc = ldc or ((C + 3) // 4) * 4
    mu0, dmu = params or logit_params(K, C)
    out = np.empty((n, K, ldc), dtype=np.float32)
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.int32)
    _lib().rkg_fill_logits(seed, n0, n, K, C, ldc, mu0, dmu, _p(yy), _p(out), _threads())
    return out


def features(seed: int, n0: int, n: int, D: int, C: int, psig_q16: int, real: bool,
             y: np.ndarray | None = None) -> np.ndarray:
    """bf16 bit patterns (uint16) of X [n][D]."""
    out = np.empty((n, D), dtype=np.uint16)
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.int32)
    _lib().rkg_fill_x(seed, n0, n, D, C, psig_q16, int(real), _p(yy), _p(out), _threads())
    return out


def weights(seed: int, K: int, C: int, D: int, flip0_q16: int, dflip_q16: int, real: bool) -> np.ndarray:
    """bf16 bit patterns (uint16) of W [K][C][D]."""
    out = np.empty((K, C, D), dtype=np.uint16)
    _lib().rkg_fill_w(seed, K, C, D, flip0_q16, dflip_q16, int(real), _p(out), _threads())
    return out


def bias(seed: int, K: int, C: int, real: bool) -> np.ndarray:
    out = np.empty((K, C), dtype=np.float32)
    _lib().rkg_fill_bias(seed, K, C, int(real), _p(out))
    return out


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ---- device fills (bench / GPU tests) ---------------------------------------------------
def _dev_lib():
    global _dev
    if _dev is None:
        L = ctypes.CDLL(build_device())
        i64, u64, i32, u32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
        L.rkg_dev_fill_labels.argtypes = [u64, i64, i64, i32, vp, vp]
        L.rkg_dev_fill_logits.argtypes = [u64, i64, i64, i32, i32, i32, i64, i64, vp, vp, vp]
        L.rkg_dev_fill_x.argtypes = [u64, i64, i64, i32, i32, u32, i32, vp, vp, vp]
        for f in (L.rkg_dev_fill_labels, L.rkg_dev_fill_logits, L.rkg_dev_fill_x):
            f.restype = ctypes.c_int
        _dev = L
    return _dev


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"device generator failed: cuda error {rc}")


def dev_labels(seed, n0, n, C, out_ptr, stream=0):
    _chk(_dev_lib().rkg_dev_fill_labels(seed, n0, n, C, out_ptr, stream))


def dev_logits(seed, n0, n, K, C, ldc, out_ptr, labels_ptr=None, params=None, stream=0):
    mu0, dmu = params or logit_params(K, C)
    _chk(_dev_lib().rkg_dev_fill_logits(seed, n0, n, K, C, ldc, mu0, dmu, labels_ptr, out_ptr, stream))


def dev_features(seed, n0, n, D, C, psig_q16, real, out_ptr, labels_ptr=None, stream=0):
    _chk(_dev_lib().rkg_dev_fill_x(seed, n0, n, D, C, psig_q16, int(real), labels_ptr, out_ptr, stream))
