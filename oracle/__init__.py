"""ORACLE package -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product (``paper_1402_5287_b200``)
never imports it, and it never imports the product.

* ``hk_oracle.c`` -- plain C schoolbook big-integer matvec (the definition written out,
  PAPER.md P:50-90), threaded over output rows; loaded with ctypes from
  ``oracle/libhk_oracle.so`` (built by ``build_oracle()`` / ``__graft_entry__.build()``).
* ``bruteforce.py`` -- Python-int dense-matrix brute force that pins the C oracle.

Parity status: every function here is pinned by tests/test_oracle_pins.py (brute force,
closed forms, structural identities from the paper, modular eigen-structure).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hk_oracle.c")
_LIB = os.path.join(_HERE, "libhk_oracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile hk_oracle.c with gcc (plain C11, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        f = lib.hk_oracle_matvec
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_int]
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def matvec(kind: int, P: int, a_mag, a_sign, x_mag, x_sign, rows=None, m=None, threads=None):
    """Exact y rows (sign-magnitude, Ly = 2L+1 limbs) of the kind's matvec.

    kind 0 Hankel (m x n window if ``m`` given: a has m+n-1 entries), 1 Toeplitz, 2 circulant.
    ``rows``: 0-based output rows to compute (default: all).  Returns (y_mag, y_sign).
    """
    lib = _load()
    n = int(x_mag.shape[0])
    m = n if m is None else int(m)
    L = (P + 63) // 64
    Ly = 2 * L + 1
    a_mag = np.ascontiguousarray(a_mag, dtype=np.uint64)
    x_mag = np.ascontiguousarray(x_mag, dtype=np.uint64)
    a_sign = np.ascontiguousarray(a_sign, dtype=np.int8)
    x_sign = np.ascontiguousarray(x_sign, dtype=np.int8)
    assert a_mag.shape[1] == L and x_mag.shape[1] == L
    rows = np.arange(m, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    y_mag = np.zeros((len(rows), Ly), dtype=np.uint64)
    y_sign = np.zeros(len(rows), dtype=np.int8)
    rc = lib.hk_oracle_matvec(int(kind), m, n, int(P), a_mag.ctypes.data, a_sign.ctypes.data,
                              x_mag.ctypes.data, x_sign.ctypes.data, rows.ctypes.data,
                              len(rows), y_mag.ctypes.data, y_sign.ctypes.data,
                              int(threads or default_threads()))
    if rc != 0:
        raise ValueError(f"hk_oracle_matvec failed: {rc}")
    return y_mag, y_sign
