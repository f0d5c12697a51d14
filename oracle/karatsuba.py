"""Algorithm 1 of the paper, literally, over Python ints -- ORACLE side, TEST INFRASTRUCTURE ONLY.

PAPER.md P:220-249 ("Calculation of the product of a Hankel matrix by a vector"), with the
readings of DESIGN.md: d and e have 2m-1 and 2m1-1 entries (steps 4 and 6, R15); n = 1 returns
a1 x1 and the three recursive calls are step 7 (R16).  Multiplications and additions of ring
elements are counted as the algorithm performs them (steps 1, 3-6, 8), so the paper's operation
counts can be checked against the literal recursion.
"""
from __future__ import annotations


class Counter:
    def __init__(self):
        self.mults = 0
        self.adds = 0


def split(a: list[int], x: list[int], ctr: Counter | None = None):
    """Steps 2-6: auxiliary vectors; 1-based a_1..a_{2n-1}, x_1..x_n stored 0-based;
    the conventions x_0 = x_{n+1} = 0 and a_{2n} = a_{2n+1} = 0 apply."""
    n = len(x)
    m = (n + 1) // 2
    m1 = (n + 2) // 2

    def A(k):  # a_k, 1-based, zero outside 1..2n-1
        return a[k - 1] if 1 <= k <= 2 * n - 1 else 0

    def X(k):  # x_k, 1-based, zero outside 1..n
        return x[k - 1] if 1 <= k <= n else 0

    f = [X(2 * i - 1) - X(2 * i) for i in range(1, m + 1)]           # step 3
    h = [X(2 * i - 1) for i in range(1, m + 1)]
    c = [A(2 * i - 1) + A(2 * i) for i in range(1, 2 * m)]           # step 4
    d = [A(2 * i) for i in range(1, 2 * m)]
    g = [X(2 * i - 2) - X(2 * i - 1) for i in range(1, m1 + 1)]      # step 5
    e = [A(2 * i - 1) for i in range(1, 2 * m1)]                     # step 6
    if ctr is not None:
        ctr.adds += len(f) + len(c) + len(g)
    return m, m1, c, d, e, f, g, h


def merge(p: list[int], q: list[int], r: list[int], n: int, ctr: Counter | None = None):
    """Step 8: y_{2i-1} = p_i - q_i, y_{2i} = p_i + r_i if 2i <= n."""
    m = (n + 1) // 2
    y = [0] * n
    for i in range(1, m + 1):
        y[2 * i - 2] = p[i - 1] - q[i - 1]
        if ctr is not None:
            ctr.adds += 1
        if 2 * i <= n:
            y[2 * i - 1] = p[i - 1] + r[i - 1]
            if ctr is not None:
                ctr.adds += 1
    return y


def algorithm1(a: list[int], x: list[int], ctr: Counter | None = None, cutoff: int = 2):
    """y = A_H x by Algorithm 1; cutoff = 2 is the paper's base case (step 1)."""
    n = len(x)
    assert len(a) == 2 * n - 1
    if n == 1:  # R16: not in the paper's listing
        if ctr is not None:
            ctr.mults += 1
        return [a[0] * x[0]]
    if n <= cutoff:
        if n == 2:  # step 1 explicit formula
            if ctr is not None:
                ctr.mults += 4
                ctr.adds += 2
            return [a[0] * x[0] + a[1] * x[1], a[1] * x[0] + a[2] * x[1]]
        if ctr is not None:
            ctr.mults += n * n
            ctr.adds += n * (n - 1)
        return [sum(a[i + j] * x[j] for j in range(n)) for i in range(n)]
    m, m1, c, d, e, f, g, h = split(a, x, ctr)
    p = algorithm1(c, h, ctr, cutoff)      # step 7.1
    q = algorithm1(d, f, ctr, cutoff)      # step 7.2
    r = algorithm1(e, g, ctr, cutoff)      # step 7.3
    return merge(p, q, r, n, ctr)


def single_level(a: list[int], x: list[int], ctr: Counter | None = None):
    """Depth-1 scheme of P:188-215: p = C h, q = D f, r = E g by schoolbook, then merge."""
    n = len(x)
    m, m1, c, d, e, f, g, h = split(a, x, ctr)

    def school(aa, xx):
        k = len(xx)
        if ctr is not None:
            ctr.mults += k * k
        return [sum(aa[i + j] * xx[j] for j in range(k)) for i in range(k)]

    return merge(school(c, h), school(d, f), school(e, g), n, ctr)
