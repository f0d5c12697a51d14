"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): F4 rounding of exact products.

SURVEY.md 8(f) F4 / DESIGN.md reading R23: the rounded product returns y to the input format,
y_i = m_i 2^-P with m_i = round_half_even(Y_i / 2^P), where Y_i is the exact integer product
(scale 2^-2P) -- i.e. the exact y rounded to P fractional bits, ties to even, sign-symmetric.
Written with Python ints straight from that definition; pinned against Python's own
round(Fraction) (round-half-even) in tests/test_oracle_pins.py."""
from __future__ import annotations

import numpy as np


def limbs_to_int(row) -> int:
    v = 0
    for k, w in enumerate(row):
        v |= int(w) << (64 * k)
    return v


def int_to_limbs(v: int, n: int) -> list[int]:
    assert 0 <= v < 1 << (64 * n)
    return [(v >> (64 * k)) & ((1 << 64) - 1) for k in range(n)]


def round_half_even_int(Y: int, P: int) -> int:
    """round(Y / 2^P), ties to the even integer (P >= 1)."""
    q, r = divmod(abs(Y), 1 << P)
    half = 1 << (P - 1)
    if r > half or (r == half and q % 2 == 1):
        q += 1
    return -q if Y < 0 else q


def round_rows(y_mag, y_sign, P: int):
    """Exact sign-magnitude rows (Ly = 2L+1 limbs) -> rounded rows (L+1 limbs, sign 0 iff zero)."""
    L = (P + 63) // 64
    out_m = np.zeros((y_mag.shape[0], L + 1), dtype=np.uint64)
    out_s = np.zeros(y_mag.shape[0], dtype=np.int8)
    for i in range(y_mag.shape[0]):
        Y = limbs_to_int(y_mag[i]) * int(y_sign[i])
        q = round_half_even_int(Y, P)
        out_m[i] = int_to_limbs(abs(q), L + 1)
        out_s[i] = (q > 0) - (q < 0)
    return out_m, out_s
