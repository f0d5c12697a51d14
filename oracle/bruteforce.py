"""Brute-force reference with Python integers -- ORACLE side, TEST INFRASTRUCTURE ONLY.

An independent second implementation used to pin the C oracle (``hk_oracle.c``): it
materialises the dense matrices exactly as the paper displays them and multiplies them with
arbitrary-precision Python ints.  Only for tiny n.  Shares nothing with the CUDA path.

  Hankel    A_H[i][j] = a_{i+j-1}           PAPER.md P:50-60 (Eq. AH)
  Toeplitz  A_T[i][j] = a_{n-i+j}           PAPER.md P:63-72 (Eq. AT)
  Circulant A_C[i][j] = a_{((i-j) mod n)+1} PAPER.md P:74-83 (first column a_1..a_n)
"""
from __future__ import annotations

import numpy as np


def to_ints(mag: np.ndarray, sign: np.ndarray) -> list[int]:
    """Sign-magnitude limb rows -> Python ints (mantissas; value = int * 2^-P)."""
    out = []
    for r in range(mag.shape[0]):
        v = int.from_bytes(np.ascontiguousarray(mag[r]).astype("<u8").tobytes(), "little")
        out.append(int(sign[r]) * v)
    return out


def from_ints(vals, nlimbs: int) -> tuple[np.ndarray, np.ndarray]:
    mag = np.zeros((len(vals), nlimbs), dtype=np.uint64)
    sign = np.zeros(len(vals), dtype=np.int8)
    for r, v in enumerate(vals):
        v = int(v)
        sign[r] = (v > 0) - (v < 0)
        b = abs(v).to_bytes(8 * nlimbs, "little")  # raises if it does not fit
        mag[r] = np.frombuffer(b, dtype="<u8")
    return mag, sign


def dense_matrix(kind: int, a: list[int], n: int, m: int | None = None) -> list[list[int]]:
    """The dense matrix of the paper's displays (1-based formulas, 0-based storage)."""
    m = n if m is None else m
    A = [[0] * n for _ in range(m)]
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            if kind == 0:
                A[i - 1][j - 1] = a[(i + j - 1) - 1]
            elif kind == 1:
                A[i - 1][j - 1] = a[(n - i + j) - 1]
            else:
                A[i - 1][j - 1] = a[((i - j) % n + 1) - 1]
    return A


def matvec_ints(kind: int, a: list[int], x: list[int], m: int | None = None) -> list[int]:
    n = len(x)
    A = dense_matrix(kind, a, n, m)
    return [sum(Ai[j] * x[j] for j in range(n)) for Ai in A]


def matvec(kind, P, a_mag, a_sign, x_mag, x_sign, m=None):
    """Boundary-layout in, boundary-layout out (Ly = 2L+1 limbs)."""
    L = (P + 63) // 64
    y = matvec_ints(kind, to_ints(a_mag, a_sign), to_ints(x_mag, x_sign), m)
    return from_ints(y, 2 * L + 1)
