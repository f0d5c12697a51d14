"""Modular fingerprints: Y mod q for every output row, computed from A mod q and X mod q
(test-side property check, valid at any size: reduction mod q is a ring homomorphism, so
(sum_j A_{idx(i,j)} X_j) mod q = sum_j (A mod q)(X mod q) mod q)."""
from __future__ import annotations

import numpy as np

QS = (16777213, 16777199, 16777183)  # primes < 2^24: products < 2^48, sums stay in int64


def residues(mag: np.ndarray, sign: np.ndarray, q: int) -> np.ndarray:
    L = mag.shape[1]
    w = np.array([pow(2, 64 * u, q) for u in range(L)], dtype=np.int64)
    r = (mag % np.uint64(q)).astype(np.int64)
    acc = np.zeros(mag.shape[0], dtype=np.int64)
    for u0 in range(0, L, 256):  # chunk so sums stay < 2^63
        acc = (acc + (r[:, u0:u0 + 256] @ w[u0:u0 + 256]) % q) % q
    return (acc * sign.astype(np.int64)) % q


def expected(kind: int, a_mag, a_sign, x_mag, x_sign, q: int, m=None) -> np.ndarray:
    a = residues(a_mag, a_sign, q)
    x = residues(x_mag, x_sign, q)
    n = x.shape[0]
    m = n if m is None else m
    if kind == 2:
        z = np.convolve(a, x) % q if n > 1 else (a * x) % q
        y = z[:n].copy()
        y[: n - 1] = (y[: n - 1] + z[n:2 * n - 1]) % q
        return y % q
    # Hankel rows i = 0..m-1: sum_j a[i+j] x[j] = full convolution with reversed x at n-1+i
    # (chunked over j so partial sums stay below 2^63)
    acc = np.zeros(m, dtype=np.int64)
    for j0 in range(0, n, 4096):
        xs = x[j0:j0 + 4096]
        z = np.convolve(a[j0:j0 + m + len(xs) - 1], xs[::-1]) % q
        acc = (acc + z[len(xs) - 1: len(xs) - 1 + m]) % q
    return acc[::-1].copy() if kind == 1 else acc


def check(kind, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, m=None, qs=QS) -> None:
    for q in qs:
        got = residues(y_mag, y_sign, q)
        want = expected(kind, a_mag, a_sign, x_mag, x_sign, q, m=m)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, f"fingerprint mod {q} differs in {bad.size} rows, first {bad[:8]}"
