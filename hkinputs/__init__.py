"""Seeded synthetic inputs for the multiprecision Hankel / Toeplitz / circulant matvec.

This module is shared by the oracle side (``oracle/``, ``tests/``) and the product side
(``bench.py``, the GPU tests).  It holds NONE of the method's arithmetic: it only draws
integer mantissas and signs in the boundary layout and knows the five BASELINE configs.

Boundary layout ("a = B0 * sum_k B^k a_k", B = 2^64, B0 = 2^-P; DESIGN.md
reading R5-R8):
  * a vector of ``count`` numbers is ``mag: uint64[count][L]`` (limb 0 least significant,
    L = ceil(P/64)) plus ``sign: int8[count]`` in {-1, 0, +1};
  * value = sign * mag * 2^-P; ``sign == 0`` iff ``mag == 0``; bits >= P are zero.

Word generator: SplitMix64's output function (Steele, Lea & Flood 2014) applied to the
counter ``c = ((seed*4 + stream) * 2^32 + entry) * 2^12 + word`` (mod 2^64); the mixed value
is ``mix((c + 1) * 0x9E3779B97F4A7C15)``.  Stream 0 draws ``a`` (or ``c``), stream 1 draws
``x``.  Words 0..L-1 are the magnitude (top limb masked to P - 64(L-1) bits), word L is the
sign word.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

HANKEL, TOEPLITZ, CIRCULANT = 0, 1, 2
KIND_NAMES = {HANKEL: "hankel", TOEPLITZ: "toeplitz", CIRCULANT: "circulant"}


def n_limbs(P: int) -> int:
    """L = ceil(P/64): 64-bit limbs per input mantissa (l = ceil(b / log2 B))."""
    return (P + 63) // 64


def n_out_limbs(P: int) -> int:
    """Ly = 2L + 1 limbs per exact output (|Y| < n (2^P-1)^2 < 2^(128 L + 63))."""
    return 2 * n_limbs(P) + 1


def a_count(kind: int, n: int, m: int | None = None) -> int:
    """Number of entries of the defining vector: 2n-1 (Hankel/Toeplitz), n (circulant,
    P:74-83), m+n-1 for an m x n rectangular Hankel window (row-block shard)."""
    if kind == CIRCULANT:
        return n
    return (m if m is not None else n) + n - 1


def splitmix64(counter: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (counter.astype(np.uint64) + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def raw_words(seed: int, stream: int, count: int, nwords: int) -> np.ndarray:
    """uint64[count][nwords] of SplitMix64 words for (seed, stream)."""
    if nwords > 4096:
        raise ValueError("at most 4096 words per entry")
    with np.errstate(over="ignore"):
        base = np.uint64(((seed * 4 + stream) & 0xFFFFFFFF) << 44 & 0xFFFFFFFFFFFFFFFF)
        e = np.arange(count, dtype=np.uint64)[:, None] << np.uint64(12)
        w = np.arange(nwords, dtype=np.uint64)[None, :]
        return splitmix64(base + e + w)


def top_mask(P: int) -> np.uint64:
    rem = P - 64 * (n_limbs(P) - 1)
    return np.uint64((1 << rem) - 1) if rem < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)


def _canon(mag: np.ndarray, sign: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    nz = mag.any(axis=1)
    sign = np.where(nz, sign, 0).astype(np.int8)
    return np.ascontiguousarray(mag), np.ascontiguousarray(sign)


def uniform(seed: int, stream: int, count: int, P: int) -> tuple[np.ndarray, np.ndarray]:
    """BASELINE configs[0..3] 'uniform signed': P random magnitude bits and an independent
    sign bit; magnitude 0 -> sign 0 (reading R8: -2^P is not representable)."""
    L = n_limbs(P)
    w = raw_words(seed, stream, count, L + 1)
    mag = w[:, :L].copy()
    mag[:, L - 1] &= top_mask(P)
    sign = np.where((w[:, L] & np.uint64(1)) != 0, -1, 1).astype(np.int8)
    return _canon(mag, sign)


def carry_stress(seed: int, stream: int, count: int, P: int) -> tuple[np.ndarray, np.ndarray]:
    """BASELINE configs[4] 'carry-stress' (reading R20): entry e even -> magnitude
    2^P-1 with sign (-1)^(e/2); entry e odd -> bit 1 of its sign word selects zero (0) or a
    uniform random magnitude (1) whose sign is bit 0."""
    L = n_limbs(P)
    w = raw_words(seed, stream, count, L + 1)
    mag = w[:, :L].copy()
    mag[:, L - 1] &= top_mask(P)
    sign = np.where((w[:, L] & np.uint64(1)) != 0, -1, 1).astype(np.int8)
    e = np.arange(count)
    even = (e % 2) == 0
    mag[even, :] = np.uint64(0xFFFFFFFFFFFFFFFF)
    mag[even, L - 1] = top_mask(P)
    sign[even] = np.where((e[even] // 2) % 2 == 0, 1, -1)
    zero_odd = (~even) & ((w[:, L] & np.uint64(2)) == 0)
    mag[zero_odd, :] = 0
    return _canon(mag, sign)


def max_magnitude(count: int, P: int, signs=None) -> tuple[np.ndarray, np.ndarray]:
    """Every magnitude 2^P-1; ``signs`` broadcast (default all +1)."""
    L = n_limbs(P)
    mag = np.full((count, L), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    mag[:, L - 1] = top_mask(P)
    sign = np.ones(count, dtype=np.int8) if signs is None else np.broadcast_to(
        np.asarray(signs, dtype=np.int8), (count,)).copy()
    return _canon(mag, sign)


def small_ints(values, P: int) -> tuple[np.ndarray, np.ndarray]:
    """Mantissas given as Python ints with |v| < 2^P (any size)."""
    L = n_limbs(P)
    mag = np.zeros((len(values), L), dtype=np.uint64)
    sign = np.zeros(len(values), dtype=np.int8)
    for i, v in enumerate(values):
        v = int(v)
        if abs(v) >> P:
            raise ValueError("|v| >= 2^P")
        sign[i] = (v > 0) - (v < 0)
        m = abs(v)
        for k in range(L):
            mag[i, k] = (m >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
    return _canon(mag, sign)


def zeros(count: int, P: int) -> tuple[np.ndarray, np.ndarray]:
    return (np.zeros((count, n_limbs(P)), dtype=np.uint64), np.zeros(count, dtype=np.int8))


RECIPES = {"uniform": uniform, "carry_stress": carry_stress}

# BASELINE.json configs (C1..C5).  C5 has two entry points (Toeplitz and circulant).
CONFIGS = {
    "C1": dict(kind=HANKEL, n=64, P=3328, seed=0, recipe="uniform"),
    "C2": dict(kind=HANKEL, n=1024, P=33216, seed=1, recipe="uniform"),
    "C3": dict(kind=HANKEL, n=8000, P=33216, seed=2, recipe="uniform"),
    "C4": dict(kind=HANKEL, n=16384, P=33216, seed=3, recipe="uniform"),
    "C5T": dict(kind=TOEPLITZ, n=4096, P=16608, seed=4, recipe="carry_stress"),
    "C5C": dict(kind=CIRCULANT, n=4096, P=16608, seed=4, recipe="carry_stress"),
}


def make_inputs(kind: int, n: int, P: int, seed: int, recipe: str = "uniform", m: int | None = None):
    """(a_mag, a_sign, x_mag, x_sign) for a kind/n/P/seed/recipe (a: stream 0, x: stream 1)."""
    gen = RECIPES[recipe]
    a = gen(seed, 0, a_count(kind, n, m), P)
    x = gen(seed, 1, n, P)
    return a[0], a[1], x[0], x[1]


def config_inputs(name: str):
    c = CONFIGS[name]
    return make_inputs(c["kind"], c["n"], c["P"], c["seed"], c["recipe"])
