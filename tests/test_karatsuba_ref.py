"""Pins for the literal Algorithm 1 reference (oracle/karatsuba.py), CPU only."""
import random

import pytest

from oracle import bruteforce as bf
from oracle import karatsuba as ka


def rand_ints(rng, k, bits=200):
    return [rng.getrandbits(bits) * (1 if rng.random() < 0.5 else -1) for _ in range(k)]


@pytest.mark.parametrize("cutoff", [2, 4, 8])
def test_algorithm1_equals_schoolbook(cutoff):
    rng = random.Random(cutoff)
    for n in list(range(1, 41)) + [64, 100, 127, 128, 129]:
        a = rand_ints(rng, 2 * n - 1)
        x = rand_ints(rng, n)
        assert ka.algorithm1(a, x, cutoff=cutoff) == bf.matvec_ints(0, a, x), (n, cutoff)


def test_single_level_equals_schoolbook():
    rng = random.Random(3)
    for n in range(2, 30):
        a = rand_ints(rng, 2 * n - 1)
        x = rand_ints(rng, n)
        assert ka.single_level(a, x) == bf.matvec_ints(0, a, x)


def test_two_row_identity():
    """C = (a_i + a_{i+1}) x_i, D = a_{i+1}(x_i - x_{i+1}), E = a_i(x_{i-1} - x_i);
    the two rows a_i x_i + a_{i+1} x_{i+1} and a_i x_{i-1} + a_{i+1} x_i are C - D and C + E."""
    rng = random.Random(4)
    for _ in range(100):
        ai, ai1, xm1, xi, xi1 = (rng.getrandbits(300) - (1 << 299) for _ in range(5))
        C = (ai + ai1) * xi
        D = ai1 * (xi - xi1)
        E = ai * (xm1 - xi)
        assert C - D == ai * xi + ai1 * xi1
        assert C + E == ai * xm1 + ai1 * xi


def test_split_examples_spec():
    """SPEC.md S:389-390 (hand application of steps 2-6 with padding)."""
    a = [11, 12, 13, 14, 15]  # a1..a5, n = 3
    x = [21, 22, 23]
    m, m1, c, d, e, f, g, h = ka.split(a, x)
    assert (m, m1) == (2, 2)
    assert c == [11 + 12, 13 + 14, 15] and d == [12, 14, 0] and e == [11, 13, 15]
    assert f == [21 - 22, 23] and h == [21, 23] and g == [-21, 22 - 23]
    a = [1, 2, 3, 4, 5, 6, 7]  # n = 4
    x = [8, 9, 10, 11]
    m, m1, c, d, e, f, g, h = ka.split(a, x)
    assert (m, m1) == (2, 3)
    assert e == [1, 3, 5, 7, 0] and g == [-8, 9 - 10, 11]


def test_merge_example_spec():
    """SPEC.md S:398 / Algorithm 1 step 8 at n = 3 and n = 4."""
    assert ka.merge([1, 2], [3, 4], [5, 6], 3) == [1 - 3, 1 + 5, 2 - 4]
    assert ka.merge([1, 2], [3, 4], [5, 6], 4) == [1 - 3, 1 + 5, 2 - 4, 2 + 6]


def test_base_case_and_recurrence_counts():
    """Step 1: n = 2 costs 4 multiplications; the recursion performs
    M(n) = 2 M(m) + M(m1) (three calls on sizes m, m, m1)."""
    ctr = ka.Counter()
    ka.algorithm1([1, 2, 3], [4, 5], ctr)
    assert ctr.mults == 4
    memo = {1: 1, 2: 4}

    def M(n):
        if n not in memo:
            memo[n] = 2 * M((n + 1) // 2) + M((n + 2) // 2)
        return memo[n]

    rng = random.Random(5)
    for n in [3, 4, 5, 7, 8, 16, 33, 64, 100]:
        ctr = ka.Counter()
        ka.algorithm1(rand_ints(rng, 2 * n - 1, 8), rand_ints(rng, n, 8), ctr)
        assert ctr.mults == M(n), n
    # Theta(n^log2 3): the ratio M(2n)/M(n) tends to 3
    assert abs(M(1 << 12) / M(1 << 11) - 3) < 0.05


def test_single_level_mult_count():
    """Depth-1 scheme: 2 m^2 + m1^2 multiplications, <= 3 m1^2."""
    for n in range(2, 40):
        ctr = ka.Counter()
        ka.single_level(list(range(2 * n - 1)), list(range(n)), ctr)
        m, m1 = (n + 1) // 2, (n + 2) // 2
        assert ctr.mults == 2 * m * m + m1 * m1 <= 3 * m1 * m1
