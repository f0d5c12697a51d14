"""Pins for the oracle (CPU only): the C oracle and the Python-int brute force are checked
against hand-derived golden vectors, closed forms, each other, and structural identities the
paper states (Toeplitz <-> Hankel by row reversal P:73; circulant embedding P:73-85) plus
mathematical invariants (symmetry, linearity, exact circulant eigen-structure mod q)."""
import json
import os
import random

import numpy as np
import pytest

import hkinputs as gen
import oracle
from oracle import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden", "vectors.json")


def _ints(mag, sign):
    return bf.to_ints(mag, sign)


def _rand_vals(rng, count, P, bits=None):
    bits = P if bits is None else bits
    out = []
    for _ in range(count):
        r = rng.random()
        if r < 0.1:
            v = 0
        elif r < 0.25:
            v = (1 << bits) - 1
        else:
            v = rng.getrandbits(bits)
        out.append(-v if rng.random() < 0.5 else v)
    return out


def _oracle_ints(kind, P, a, x, m=None, rows=None):
    am, asg = gen.small_ints(a, P)
    xm, xsg = gen.small_ints(x, P)
    ym, ys = oracle.matvec(kind, P, am, asg, xm, xsg, rows=rows, m=m, threads=2)
    return _ints(ym, ys), ym, ys


# ---------------------------------------------------------------------------------------------
def test_golden_vectors():
    doc = json.load(open(GOLD))
    for g in doc["vectors"]:
        P, kind = g["P"], g["kind"]
        a = [int(v, 0) if isinstance(v, str) else v for v in g["a"]]
        x = [int(v, 0) if isinstance(v, str) else v for v in g["x"]]
        am, asg = gen.small_ints(a, P)
        xm, xsg = gen.small_ints(x, P)
        want_sign = np.array([row[0] for row in g["y"]], dtype=np.int8)
        want_mag = np.array([[int(h, 16) for h in row[1]] for row in g["y"]], dtype=np.uint64)
        ym, ys = oracle.matvec(kind, P, am, asg, xm, xsg, threads=1)
        assert np.array_equal(ym, want_mag) and np.array_equal(ys, want_sign), g["id"]
        bm, bs = bf.matvec(kind, P, am, asg, xm, xsg)
        assert np.array_equal(bm, want_mag) and np.array_equal(bs, want_sign), g["id"]


@pytest.mark.parametrize("P", [1, 2, 63, 64, 65, 127, 128, 129, 200, 3328])
def test_c_oracle_vs_bruteforce(P):
    rng = random.Random(1000 + P)
    ns = [1, 2, 3, 4, 5, 7, 8, 13, 16, 24] if P <= 200 else [1, 2, 3, 5, 8]
    for n in ns:
        for kind in (0, 1, 2):
            a = _rand_vals(rng, gen.a_count(kind, n), P)
            x = _rand_vals(rng, n, P)
            got, ym, ys = _oracle_ints(kind, P, a, x)
            assert got == bf.matvec_ints(kind, a, x), (P, n, kind)
            # canonical form: sign 0 iff zero, unused limbs zero by construction of ints
            assert np.all((ys == 0) == (~ym.any(axis=1)))
    # rectangular Hankel windows (row-block shards)
    for (m, n) in [(1, 5), (3, 7), (6, 2), (9, 9)]:
        a = _rand_vals(rng, m + n - 1, P)
        x = _rand_vals(rng, n, P)
        got, _, _ = _oracle_ints(0, P, a, x, m=m)
        assert got == bf.matvec_ints(0, a, x, m=m)


def test_row_subset_matches_full():
    am, asg, xm, xsg = gen.make_inputs(0, 37, 700, seed=9)
    full_m, full_s = oracle.matvec(0, 700, am, asg, xm, xsg, threads=3)
    rows = np.array([36, 0, 17, 5], dtype=np.int64)
    sub_m, sub_s = oracle.matvec(0, 700, am, asg, xm, xsg, rows=rows, threads=2)
    assert np.array_equal(sub_m, full_m[rows]) and np.array_equal(sub_s, full_s[rows])


# ---------------------------------------------------------------------------------------------
# closed forms
@pytest.mark.parametrize("n,P", [(1, 64), (5, 65), (16, 128), (33, 1000), (64, 3328)])
def test_closed_form_max_magnitude(n, P):
    """All entries +(2^P-1): Y_i = n (2^P-1)^2 (largest output; exercises the top limb)."""
    M = (1 << P) - 1
    for kind in (0, 1, 2):
        am, asg = gen.max_magnitude(gen.a_count(kind, n), P)
        xm, xsg = gen.max_magnitude(n, P)
        ym, ys = oracle.matvec(kind, P, am, asg, xm, xsg, threads=2)
        assert _ints(ym, ys) == [n * M * M] * n


@pytest.mark.parametrize("n", [1, 2, 3, 10, 31, 64])
def test_closed_form_alternating(n):
    """a_k = 2^P-1, x_j = (-1)^j (2^P-1): Y_i = 0 for even n, -(2^P-1)^2 for odd n."""
    P = 190
    M = (1 << P) - 1
    am, asg = gen.max_magnitude(2 * n - 1, P)
    xm, xsg = gen.max_magnitude(n, P, signs=[(-1) ** j for j in range(1, n + 1)])
    ym, ys = oracle.matvec(0, P, am, asg, xm, xsg, threads=2)
    want = 0 if n % 2 == 0 else -M * M
    assert _ints(ym, ys) == [want] * n
    if want == 0:
        assert not ys.any() and not ym.any()


@pytest.mark.parametrize("n", [1, 4, 9, 50])
def test_closed_form_index_sum(n):
    """a_k = k, x_j = 1: Y_i = sum_j (i+j-1) = n(i-1) + n(n+1)/2 (pins the Hankel index)."""
    P = 64
    a = list(range(1, 2 * n))
    x = [1] * n
    got, _, _ = _oracle_ints(0, P, a, x)
    assert got == [n * (i - 1) + n * (n + 1) // 2 for i in range(1, n + 1)]


def test_zero_vector():
    am, asg, _, _ = gen.make_inputs(0, 20, 300, seed=3)
    xm, xsg = gen.zeros(20, 300)
    ym, ys = oracle.matvec(0, 300, am, asg, xm, xsg, threads=2)
    assert not ym.any() and not ys.any()


def test_unit_vectors_select_columns():
    """x = e_j gives y = column j: (a_j .. a_{j+n-1}) for Hankel."""
    rng = random.Random(5)
    n, P = 9, 300
    a = _rand_vals(rng, 2 * n - 1, P)
    for j in range(1, n + 1):
        x = [1 if k == j else 0 for k in range(1, n + 1)]
        got, _, _ = _oracle_ints(0, P, a, x)
        assert got == a[j - 1:j - 1 + n]


# ---------------------------------------------------------------------------------------------
# structural identities (paper) and invariants (mathematics)
@pytest.mark.parametrize("n", [1, 2, 7, 16])
def test_toeplitz_is_reversed_hankel(n):
    """a Toeplitz matrix becomes Hankel by reversing its rows."""
    am, asg, xm, xsg = gen.make_inputs(0, n, 500, seed=n)
    hm, hs = oracle.matvec(0, 500, am, asg, xm, xsg, threads=2)
    tm, ts = oracle.matvec(1, 500, am, asg, xm, xsg, threads=2)
    assert np.array_equal(tm, hm[::-1]) and np.array_equal(ts, hs[::-1])


@pytest.mark.parametrize("n", [1, 2, 5, 8])
def test_circulant_embeds_in_toeplitz(n):
    """the n x n circulant with first column c equals the Toeplitz matrix of
    t = (c_n, ..., c_1, c_n, ..., c_2)."""
    P = 400
    cm, cs, xm, xsg = gen.make_inputs(2, n, P, seed=11 + n)
    idx = list(range(n - 1, -1, -1)) + list(range(n - 1, 0, -1))
    tm_, ts_ = cm[idx], cs[idx]
    ym, ys = oracle.matvec(2, P, cm, cs, xm, xsg, threads=2)
    zm, zs = oracle.matvec(1, P, tm_, ts_, xm, xsg, threads=2)
    assert np.array_equal(ym, zm) and np.array_equal(ys, zs)


def test_circulant_is_cyclic_convolution():
    rng = random.Random(8)
    n, P = 11, 150
    c = _rand_vals(rng, n, P)
    x = _rand_vals(rng, n, P)
    got, _, _ = _oracle_ints(2, P, c, x)
    assert got == [sum(c[(i - j) % n] * x[j] for j in range(n)) for i in range(n)]


def test_hankel_symmetry():
    """A_H is symmetric: z^T (A x) = x^T (A z)."""
    P, n = 257, 12
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=21)
    zm, zs = gen.uniform(22, 1, n, P)
    y1 = _ints(*oracle.matvec(0, P, am, asg, xm, xsg, threads=2))
    y2 = _ints(*oracle.matvec(0, P, am, asg, zm, zs, threads=2))
    x = _ints(xm, xsg)
    z = _ints(zm, zs)
    assert sum(a * b for a, b in zip(z, y1)) == sum(a * b for a, b in zip(x, y2))


def test_linearity_in_x():
    """y(x + z) = y(x) + y(z) with x, z drawn at P-1 bits so x + z stays within P bits."""
    rng = random.Random(31)
    P, n = 321, 10
    for kind in (0, 1, 2):
        a = _rand_vals(rng, gen.a_count(kind, n), P)
        x = _rand_vals(rng, n, P, bits=P - 1)
        z = _rand_vals(rng, n, P, bits=P - 1)
        yx, _, _ = _oracle_ints(kind, P, a, x)
        yz, _, _ = _oracle_ints(kind, P, a, z)
        yxz, _, _ = _oracle_ints(kind, P, a, [u + v for u, v in zip(x, z)])
        assert yxz == [u + v for u, v in zip(yx, yz)]


@pytest.mark.parametrize("n", [4, 8, 16])
def test_circulant_eigenstructure_mod_q(n):
    """Exact eigen-structure of circulants mod q = 12289 (n | q-1): with v_j = w^(jk),
    (C v)_i = w^(ik) * lambda_k, lambda_k = sum_t c_t w^(-tk)  (0-based c_t = c_{t+1})."""
    q = 12289
    g = 11  # primitive root mod 12289
    w = pow(g, (q - 1) // n, q)
    P = 500
    cm, cs = gen.uniform(40 + n, 0, n, P)
    c = _ints(cm, cs)
    for k in range(n):
        v = [pow(w, j * k, q) for j in range(n)]
        vm, vs = gen.small_ints(v, P)
        y = _ints(*oracle.matvec(2, P, cm, cs, vm, vs, threads=2))
        lam = sum(c[t] * pow(w, (-t * k) % n, q) for t in range(n)) % q
        assert [yi % q for yi in y] == [(pow(w, i * k, q) * lam) % q for i in range(n)]


def test_baseline_config_c1_full_vs_bruteforce():
    """C1 (n=64, P=3328, seed 0) in full: C oracle == Python ints."""
    am, asg, xm, xsg = gen.config_inputs("C1")
    ym, ys = oracle.matvec(0, 3328, am, asg, xm, xsg)
    bm, bs = bf.matvec(0, 3328, am, asg, xm, xsg)
    assert np.array_equal(ym, bm) and np.array_equal(ys, bs)


def test_carry_stress_config_rows_vs_bruteforce():
    """C5 recipe (carry-stress) on a reduced n, both kinds: C oracle == Python ints."""
    for kind in (1, 2):
        am, asg, xm, xsg = gen.make_inputs(kind, 24, 1000, seed=4, recipe="carry_stress")
        ym, ys = oracle.matvec(kind, 1000, am, asg, xm, xsg, threads=2)
        bm, bs = bf.matvec(kind, 1000, am, asg, xm, xsg)
        assert np.array_equal(ym, bm) and np.array_equal(ys, bs)


# ---------------------------------------------------------------------------------------------
# F4 rounding (oracle/rounding.py): pinned to Python's round(Fraction), which rounds half to even
def test_round_half_even_matches_fraction_round():
    import random
    from fractions import Fraction
    from oracle import rounding as rd
    rng = random.Random(7)
    for P in (1, 2, 5, 63, 64, 65, 127, 128, 200):
        for _ in range(200):
            Y = rng.getrandbits(2 * P + 14) * rng.choice((-1, 1))
            assert rd.round_half_even_int(Y, P) == round(Fraction(Y, 1 << P))
        for k in (-5, -3, -1, 0, 1, 2, 3, 4):  # exact ties k + 1/2 and exact integers
            Yt = (2 * k + 1) << (P - 1)
            assert rd.round_half_even_int(Yt, P) == round(Fraction(Yt, 1 << P))
            assert rd.round_half_even_int(k << P, P) == k


def test_round_half_even_closed_cases():
    from oracle import rounding as rd
    assert [rd.round_half_even_int(Y, 1) for Y in (1, 3, 5, 7, -1, -3, -5)] == [0, 2, 2, 4, 0, -2, -2]
    P = 70  # increment carrying across limbs: (2^128 - 1) + 1/2 + tiny -> 2^128
    Y = ((1 << 128) - 1 << P) + (1 << (P - 1)) + 1
    assert rd.round_half_even_int(Y, P) == 1 << 128
    m, s = rd.round_rows(np.array([rd.int_to_limbs(Y, 5)], dtype=np.uint64), np.array([1], np.int8), 128)
    assert s[0] == 1 and rd.limbs_to_int(m[0]) == rd.round_half_even_int(Y, 128)
    m, s = rd.round_rows(np.array([[1, 0, 0]], dtype=np.uint64), np.array([-1], np.int8), 64)
    assert s[0] == 0 and not m.any()  # -2^-128 rounds to a canonical zero
