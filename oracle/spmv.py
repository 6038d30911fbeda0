"""Oracle: ctypes loader for spmv_ref.c + acceptance check.

Test infrastructure only (see oracle/__init__.py).  `build_oracle()` compiles the C file
with gcc; `__graft_entry__.build()` calls it ("building the checker is not using it").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spmv_ref.c")
_LIB = os.path.join(_HERE, "liboracle_spmv.so")
_lib = None

TOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}   # north_star, reading A2/O2


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", _SRC, "-o", _LIB, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_oracle())
        f = _lib.oracle_spmv_csr
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 4 + [ctypes.c_double, ctypes.c_double,
                                                                  ctypes.c_void_p, ctypes.c_void_p,
                                                                  ctypes.c_void_p, ctypes.c_int]
    return _lib


def spmv_csr(row_ptr, col, val, x, alpha=1.0, beta=0.0, y0=None, nthreads=1):
    """Returns (yref, bound) as np.longdouble arrays of length m."""
    lib = _load()
    m = row_ptr.shape[0] - 1
    rp = np.ascontiguousarray(row_ptr, np.int64)
    c = np.ascontiguousarray(col, np.int64)
    v = np.ascontiguousarray(val, np.float64)
    xx = np.ascontiguousarray(x, np.float64)
    yy = np.ascontiguousarray(y0 if y0 is not None else np.zeros(m), np.float64)
    y = np.zeros(m, np.longdouble)
    b = np.zeros(m, np.longdouble)
    lib.oracle_spmv_csr(m, rp.ctypes.data, c.ctypes.data, v.ctypes.data, xx.ctypes.data,
                        float(alpha), float(beta), yy.ctypes.data, y.ctypes.data, b.ctypes.data,
                        int(nthreads))
    return y, b


def coo_to_csr(m, row, col, val):
    """Canonical CSR (rows ascending, cols ascending) from COO triplets."""
    order = np.lexsort((col, row))
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, np.asarray(row, np.int64) + 1, 1)
    return np.cumsum(rp), np.asarray(col, np.int64)[order], np.asarray(val, np.float64)[order]


def spmv_coo(m, row, col, val, x, alpha=1.0, beta=0.0, y0=None, nthreads=1):
    rp, c, v = coo_to_csr(m, row, col, val)
    return spmv_csr(rp, c, v, x, alpha, beta, y0, nthreads)


def check(y, yref, bound, dtype, tol=None):
    """O2: |y_i - yref_i| <= tol * bound_i in long double; bound 0 => y must be +-0.
    Returns (ok, max_ratio)."""
    tol = TOL[np.dtype(dtype)] if tol is None else tol
    err = np.abs(np.asarray(y).astype(np.longdouble) - yref)
    lim = np.longdouble(tol) * bound
    ok = bool(np.all(err <= lim))
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1), np.where(err > 0, np.inf, 0))
    return ok, float(ratio.max()) if ratio.shape[0] else 0.0
