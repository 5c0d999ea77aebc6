"""ctypes wrapper of oracle/dense.c (float64 dense direct sums).  TEST INFRASTRUCTURE ONLY.

The C file is compiled on first use with plain ``gcc -O2 -fopenmp`` (no
fast-math) if ``liboracle_dense.so`` is missing or older than the source;
``__graft_entry__.build()`` also compiles it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dense.c")
_LIB = os.path.join(_HERE, "liboracle_dense.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile dense.c -> liboracle_dense.so (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            d, i32, i64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64
            P = ctypes.c_void_p
            lib.oracle_dense_apply.argtypes = [i64, i32, P, i32, P, P, i32, d, d, d, i32, P, i64, P, P, P, P, P]
            lib.oracle_dense_apply.restype = ctypes.c_int
            lib.oracle_kernel_value.argtypes = [i32, P, i32, d, i32]
            lib.oracle_kernel_value.restype = d
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def dense_apply(X, windows, family, theta, V, rows=None, ops=("K", "dell", "dsf", "dse")):
    """Dense float64 products (eqs. 2.1-2.3): returns dict op -> (len(rows) or n) x r array.

    X: n x p, windows: list of feature-index tuples (0-based), family 0 Gaussian / 1 Matern(1/2),
    theta = (sigma_f, ell, sigma_eps), V: n x r.  rows: optional int64 row subset.
    """
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    if V.ndim == 1:
        V = V[:, None]
    n, p = X.shape
    r = V.shape[1]
    feat = np.array([f for w in windows for f in w], dtype=np.int32)
    lens = np.array([len(w) for w in windows], dtype=np.int32)
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        nrows = rows.shape[0]
    else:
        nrows = n
    out = {op: np.zeros((nrows, r), dtype=np.float64) for op in ops}
    sf, ell, se = (float(t) for t in theta)
    rc = lib.oracle_dense_apply(n, p, _ptr(X), len(windows), _ptr(feat), _ptr(lens), int(family), sf, ell, se, r,
                                _ptr(V), nrows, _ptr(rows), _ptr(out.get("K")), _ptr(out.get("dell")),
                                _ptr(out.get("dsf")), _ptr(out.get("dse")))
    if rc != 0:
        raise ValueError("oracle_dense_apply rejected its arguments")
    return out


def kernel_value(family, rvec, ell, deriv=False):
    """Sub-kernel value kappa(r) (eq. 1.1 without sigma_f^2) or its ell-derivative (eq. 2.3)."""
    lib = _load()
    rv = np.ascontiguousarray(np.atleast_1d(rvec), dtype=np.float64)
    return lib.oracle_kernel_value(int(family), _ptr(rv), rv.shape[0], float(ell), int(bool(deriv)))
