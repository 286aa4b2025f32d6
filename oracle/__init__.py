"""ctypes binding of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module.  The product
path (paper_2407_07058_b200) never imports it, and it imports nothing from the
product.  See oracle.c for the paper passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-math-errno", "-mfma", "-shared", "-fPIC"]


class Stats(ctypes.Structure):
    _fields_ = [
        ("writes", ctypes.c_int64),
        ("traversed", ctypes.c_int64),
        ("t_mst", ctypes.c_double),
        ("t_sort", ctypes.c_double),
        ("t_copy", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.oracle_r1_dist2.restype = ctypes.c_float
        L.oracle_r1_dist2.argtypes = [P, P, I64]
        L.oracle_r1_weight.restype = ctypes.c_float
        L.oracle_r1_weight.argtypes = [P, P, I64]
        L.oracle_dist_f64.restype = ctypes.c_double
        L.oracle_dist_f64.argtypes = [P, P, I64]
        L.oracle_points_weights.restype = None
        L.oracle_points_weights.argtypes = [P, I64, I64, I64, I64, P]
        L.oracle_points_weights_metric.restype = None
        L.oracle_points_weights_metric.argtypes = [P, I64, I64, ctypes.c_int, I64, I64, P]
        L.oracle_metric_weight.restype = ctypes.c_float
        L.oracle_metric_weight.argtypes = [P, P, I64, ctypes.c_int]
        L.oracle_appd_points_metric.argtypes = [P, I64, I64, ctypes.c_int, P, P]
        L.oracle_prim_weights.argtypes = [P, I64, ctypes.c_int, P, P, P]
        L.oracle_prim_points.argtypes = [P, I64, I64, P, P, P]
        L.oracle_appd_weights.argtypes = [P, I64, ctypes.c_int, P, P]
        L.oracle_appd_weights_f64.argtypes = [P, I64, ctypes.c_int, P, P]
        L.oracle_prim_weights_f64.argtypes = [P, I64, ctypes.c_int, P, P, P]
        L.oracle_appd_points.argtypes = [P, I64, I64, P, P]
        L.oracle_appd_points_rows.argtypes = [P, I64, I64, I64, I64, P, P]
        L.oracle_appd_weights_rows.argtypes = [P, I64, I64, I64, P, P]
        L.oracle_floyd.argtypes = [P, I64, ctypes.c_int, P]
        L.oracle_brute.argtypes = [P, I64, ctypes.c_int, P]
        L.oracle_mst_path.argtypes = [P, I64, P]
        L.oracle_fnv1a64.restype = ctypes.c_uint64
        L.oracle_fnv1a64.argtypes = [P, I64]
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


def appd_weights(W, sense: int = 1, with_stats: bool = False):
    """Algorithm 4 on a dense symmetric fp32 weight matrix."""
    W = _f32(W)
    n = W.shape[0]
    M = np.empty((n, n), dtype=np.float32)
    st = Stats()
    _check(lib().oracle_appd_weights(_ptr(W), n, sense, _ptr(M), ctypes.byref(st)), "appd_weights")
    return (M, st.as_dict()) if with_stats else M


def appd_weights_f64(W, sense: int = 1, with_stats: bool = False):
    """NEXT-3: Algorithm 4 on a dense symmetric fp64 weight matrix, fp64 M."""
    W = np.ascontiguousarray(W, dtype=np.float64)
    n = W.shape[0]
    M = np.empty((n, n), dtype=np.float64)
    st = Stats()
    _check(lib().oracle_appd_weights_f64(_ptr(W), n, sense, _ptr(M), ctypes.byref(st)), "appd_weights_f64")
    return (M, st.as_dict()) if with_stats else M


def prim_weights_f64(W, sense: int = 1):
    """NEXT-3: Prim on an fp64 weight matrix: (eu, ev, ew) in attachment order."""
    W = np.ascontiguousarray(W, dtype=np.float64)
    n = W.shape[0]
    m = max(n - 1, 0)
    eu = np.empty(m, dtype=np.int32)
    ev = np.empty(m, dtype=np.int32)
    ew = np.empty(m, dtype=np.float64)
    _check(lib().oracle_prim_weights_f64(_ptr(W), n, sense, _ptr(eu), _ptr(ev), _ptr(ew)), "prim_weights_f64")
    return eu, ev, ew


def appd_points(X, with_stats: bool = False, metric: int = 0):
    """Algorithm 4 on the complete graph of the points X (n x d): R1 weights (metric 0),
    Manhattan (1) or Chebyshev (2) distances (NEXT-3)."""
    X = _f32(X)
    n, d = X.shape
    M = np.empty((n, n), dtype=np.float32)
    st = Stats()
    if metric == 0:
        _check(lib().oracle_appd_points(_ptr(X), n, d, _ptr(M), ctypes.byref(st)), "appd_points")
    else:
        _check(lib().oracle_appd_points_metric(_ptr(X), n, d, metric, _ptr(M), ctypes.byref(st)), "appd_points")
    return (M, st.as_dict()) if with_stats else M


def appd_points_rows(X, r0: int, R: int, with_stats: bool = False):
    """R5: rows [r0, r0+R) of the points-mode APPD."""
    X = _f32(X)
    n, d = X.shape
    M = np.empty((R, n), dtype=np.float32)
    st = Stats()
    _check(lib().oracle_appd_points_rows(_ptr(X), n, d, r0, R, _ptr(M), ctypes.byref(st)), "appd_points_rows")
    return (M, st.as_dict()) if with_stats else M


def appd_weights_rows(W, r0: int, R: int):
    W = _f32(W)
    n = W.shape[0]
    M = np.empty((R, n), dtype=np.float32)
    st = Stats()
    _check(lib().oracle_appd_weights_rows(_ptr(W), n, r0, R, _ptr(M), ctypes.byref(st)), "appd_weights_rows")
    return M


def prim_weights(W, sense: int = 1):
    W = _f32(W)
    n = W.shape[0]
    m = max(n - 1, 0)
    eu = np.empty(m, np.int32)
    ev = np.empty(m, np.int32)
    ew = np.empty(m, np.float32)
    _check(lib().oracle_prim_weights(_ptr(W), n, sense, _ptr(eu), _ptr(ev), _ptr(ew)), "prim_weights")
    return eu, ev, ew


def prim_points(X):
    X = _f32(X)
    n, d = X.shape
    m = max(n - 1, 0)
    eu = np.empty(m, np.int32)
    ev = np.empty(m, np.int32)
    ew = np.empty(m, np.float32)
    _check(lib().oracle_prim_points(_ptr(X), n, d, _ptr(eu), _ptr(ev), _ptr(ew)), "prim_points")
    return eu, ev, ew


def floyd(W, sense: int = 1):
    W = _f32(W)
    n = W.shape[0]
    M = np.empty((n, n), dtype=np.float32)
    _check(lib().oracle_floyd(_ptr(W), n, sense, _ptr(M)), "floyd")
    return M


def brute(W, sense: int = 1):
    W = _f32(W)
    n = W.shape[0]
    M = np.empty((n, n), dtype=np.float32)
    _check(lib().oracle_brute(_ptr(W), n, sense, _ptr(M)), "brute")
    return M


def mst_path(W):
    W = _f32(W)
    n = W.shape[0]
    M = np.empty((n, n), dtype=np.float32)
    _check(lib().oracle_mst_path(_ptr(W), n, _ptr(M)), "mst_path")
    return M


def r1_dist2(xi, xj) -> np.float32:
    xi, xj = _f32(xi), _f32(xj)
    return np.float32(lib().oracle_r1_dist2(_ptr(xi), _ptr(xj), xi.shape[0]))


def r1_weight(xi, xj) -> np.float32:
    xi, xj = _f32(xi), _f32(xj)
    return np.float32(lib().oracle_r1_weight(_ptr(xi), _ptr(xj), xi.shape[0]))


def dist_f64(xi, xj) -> float:
    xi, xj = _f32(xi), _f32(xj)
    return float(lib().oracle_dist_f64(_ptr(xi), _ptr(xj), xi.shape[0]))


def points_weights(X, r0: int = 0, R: int | None = None, metric: int = 0):
    """Row block [r0, r0+R) of the weight matrix (R1, or the metric of NEXT-3)."""
    X = _f32(X)
    n, d = X.shape
    R = n - r0 if R is None else R
    Wb = np.empty((R, n), dtype=np.float32)
    if metric == 0:
        lib().oracle_points_weights(_ptr(X), n, d, r0, R, _ptr(Wb))
    else:
        lib().oracle_points_weights_metric(_ptr(X), n, d, metric, r0, R, _ptr(Wb))
    return Wb


def fnv1a64(a) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().oracle_fnv1a64(_ptr(a), a.nbytes))
