"""F3 planner pins (CPU): the digit width and error bound hk_fft_plan chooses for the FP64 FFT path,
against an independent restatement of Percival's theorem in 60-digit decimal arithmetic, plus the
measured error of a plain radix-2 FP64 FFT convolution staying under that bound.

Percival, "Rapid multiplication modulo the sum and difference of highly composite numbers",
Math. Comp. 72 (2003), Thm 5.1: a length-2^k cyclic convolution z of x and y computed by radix-2
FFTs in floating point (unit roundoff e, precomputed twiddles with error b) satisfies
    |z' - z|_inf < |x|_2 |y|_2 ((1 + e)^(3k) (1 + e sqrt5)^(3k + 1) (1 + b)^(3k) - 1).
DESIGN.md reading R24: the N1 x N2 row-column transform is k = log2(N1 N2) radix-2 stages of the
same kind.  Digits are balanced, |d| <= 2^(w-1), so |a|_2 |x|_2 <= sqrt(a_count n) Ls 2^(2w-2).
PAPER.md P:119-170 (decomposition approach), P:169 (the accuracy question this answers)."""
from decimal import Decimal, getcontext

import numpy as np
import pytest

import hkinputs as gen

getcontext().prec = 60
EPS = Decimal(2) ** -53
BETA = Decimal(2) ** -52


def percival_factor(k: int) -> Decimal:
    return ((1 + EPS) ** (3 * k)) * ((1 + EPS * Decimal(5).sqrt()) ** (3 * k + 1)) * ((1 + BETA) ** (3 * k)) - 1


def log2ceil(v: int) -> int:
    return max(0, (v - 1).bit_length())


def reference_plan(kind: int, n: int, P: int, max_log_n1=15, max_log_n2=13):
    """Widest balanced digit width w whose bound is <= 0.49 (None if none fits the limits)."""
    a_count = n if kind == gen.CIRCULANT else 2 * n - 1
    if kind == gen.CIRCULANT and n & (n - 1) == 0 and n >= 32:
        lg1 = log2ceil(n)
    else:
        lg1 = max(5, log2ceil(2 * n - 1 if kind == gen.CIRCULANT else a_count))
    if lg1 > max_log_n1:
        return None
    for w in range(30, 1, -1):
        Ls = -(-P // w) + 1
        lg2 = max(5, log2ceil(2 * Ls - 1))
        if lg2 > max_log_n2:
            continue
        d = Decimal(2) ** (w - 1)
        B = (Decimal(a_count * n).sqrt() * Ls * d * d) * percival_factor(lg1 + lg2)
        if B <= Decimal("0.49") and n * Ls * d * d < Decimal(2) ** 52:
            return dict(w=w, Ls=Ls, log_n1=lg1, log_n2=lg2, bound=float(B))
    return None


CASES = [(0, 64, 3328), (1, 64, 3328), (2, 64, 3328), (0, 1024, 33216), (2, 4096, 16608),
         (0, 1, 1), (0, 2, 64), (1, 17, 1000), (2, 100, 5000), (2, 128, 700), (0, 300, 20000),
         (0, 2048, 33216), (2, 33, 65)]


@pytest.mark.parametrize("kind,n,P", CASES)
def test_planner_matches_percival(kind, n, P):
    import paper_1402_5287_b200 as hk
    ref = reference_plan(kind, n, P)
    if ref is None:
        with pytest.raises(hk.HKError):
            hk.fft_plan(kind, n, P)
        return
    got = hk.fft_plan(kind, n, P)
    assert (got["w"], got["Ls"], got["log_n1"], got["log_n2"]) == (ref["w"], ref["Ls"], ref["log_n1"], ref["log_n2"])
    assert abs(got["bound"] - ref["bound"]) <= 1e-9 * ref["bound"]
    assert got["bound"] <= 0.49


def test_bound_is_tight_in_w():
    """The chosen w is the widest: w + 1 breaks the bound or the supported lengths."""
    for kind, n, P in CASES:
        ref = reference_plan(kind, n, P)
        if ref is None or ref["w"] == 30:
            continue
        w = ref["w"] + 1
        Ls = -(-P // w) + 1
        lg2 = max(5, log2ceil(2 * Ls - 1))
        a_count = n if kind == gen.CIRCULANT else 2 * n - 1
        d = Decimal(2) ** (w - 1)
        B = Decimal(a_count * n).sqrt() * Ls * d * d * percival_factor(ref["log_n1"] + lg2)
        assert B > Decimal("0.49") or lg2 > 13 or n * Ls * d * d >= Decimal(2) ** 52


def test_baseline_configs_bound():
    """at C3 (n 8000, P 33,216) balanced 10-bit digits meet the bound (0.466
    with beta = 2^-52; 11 bits do not), C2 takes 11 bits, C4 9 bits -- a proven FP64 path exists
    for every BASELINE config, and the library plans every one of them."""
    import paper_1402_5287_b200 as hk
    expect = {"C1": 15, "C2": 11, "C3": 10, "C4": 9, "C5T": 11, "C5C": 11}
    for name, w in expect.items():
        c = gen.CONFIGS[name]
        ref = reference_plan(c["kind"], c["n"], c["P"], max_log_n1=15)
        assert ref is not None and ref["w"] == w, (name, ref)
        assert hk.fft_plan(c["kind"], c["n"], c["P"])["w"] == w
    assert abs(reference_plan(0, 8000, 33216, max_log_n1=15)["bound"] - 0.466) < 0.001


def _fft(v, inverse=False):
    """Plain iterative radix-2 complex FFT (DIT over bit-reversed input) in float64, last axis."""
    n = v.shape[-1]
    bits = n.bit_length() - 1
    idx = np.array([int(format(i, f"0{bits}b")[::-1], 2) for i in range(n)])
    a = v[..., idx].astype(np.complex128)
    h = 1
    while h < n:
        w = np.exp((2j if inverse else -2j) * np.pi * np.arange(h) / (2 * h))
        a = a.reshape(a.shape[:-1] + (n // (2 * h), 2, h))
        t = a[..., 1, :] * w
        a = np.stack([a[..., 0, :] + t, a[..., 0, :] - t], axis=-2).reshape(a.shape[:-3] + (n,))
        h *= 2
    return a


def test_radix2_fft_error_below_bound():
    """Max-magnitude balanced digits (the bound's worst case for the norms) convolved by a plain
    radix-2 FP64 FFT: the error against the exact integer convolution is below the bound."""
    rng = np.random.default_rng(5)
    n, P = 32, 400
    ref = reference_plan(0, n, P)
    w, Ls = ref["w"], ref["Ls"]
    N1, N2 = 1 << ref["log_n1"], 1 << ref["log_n2"]
    d = 2 ** (w - 1)
    A = np.zeros((N1, N2), dtype=np.int64)
    X = np.zeros((N1, N2), dtype=np.int64)
    A[: 2 * n - 1, :Ls] = rng.choice([-d, d], size=(2 * n - 1, Ls))
    X[:n, :Ls] = rng.choice([-d, d], size=(n, Ls))

    def fft2(M, inv=False):
        return _fft(_fft(M, inv).swapaxes(0, 1), inv).swapaxes(0, 1)

    Z = fft2(fft2(A) * fft2(X), True).real / (N1 * N2)
    exact = np.zeros((N1, N2), dtype=np.int64)  # cyclic in the row index, linear in the digit index
    for i in np.nonzero(A.any(axis=1))[0]:
        for j in np.nonzero(X.any(axis=1))[0]:
            exact[(i + j) % N1] += np.convolve(A[i, :Ls], X[j, :Ls], mode="full").tolist() + [0] * (N2 - 2 * Ls + 1)
    err = np.abs(Z - exact).max()
    assert err < ref["bound"] < 0.5, (err, ref["bound"])


def forced_bound(kind: int, n: int, P: int, w: int):
    """Percival's bound at a FORCED digit width w (the accuracy study's plans), 60-digit decimal."""
    a_count = n if kind == gen.CIRCULANT else 2 * n - 1
    if kind == gen.CIRCULANT and n & (n - 1) == 0 and n >= 32:
        lg1 = log2ceil(n)
    else:
        lg1 = max(5, log2ceil(2 * n - 1 if kind == gen.CIRCULANT else a_count))
    Ls = -(-P // w) + 1
    lg2 = max(5, log2ceil(2 * Ls - 1))
    d = Decimal(2) ** (w - 1)
    return dict(Ls=Ls, log_n1=lg1, log_n2=lg2,
                bound=float(Decimal(a_count * n).sqrt() * Ls * d * d * percival_factor(lg1 + lg2)),
                fits=lg2 <= 13 and n * Ls * d * d < Decimal(2) ** 62)


def test_forced_width_plans():
    """hk_fft_plan_w (F3 accuracy study): w = 0 is the proven plan; a forced w reports that width's
    Percival bound (a restatement of the theorem, 60 digits), past 1/2 for widths wider than the
    proven one, and refuses widths whose digit FFT or coefficients do not fit."""
    import paper_1402_5287_b200 as hk
    for kind, n, P in [(0, 8000, 33216), (0, 1024, 33216), (1, 4096, 16608), (2, 64, 3328)]:
        proven = hk.fft_plan(kind, n, P)
        assert hk.fft_plan(kind, n, P, w=0) == proven
        assert hk.fft_plan(kind, n, P, w=proven["w"]) == proven
        prev = 0.0
        for w in range(2, 31):
            ref = forced_bound(kind, n, P, w)
            if not ref["fits"]:
                with pytest.raises(hk.HKError):
                    hk.fft_plan(kind, n, P, w=w)
                continue
            got = hk.fft_plan(kind, n, P, w=w)
            assert (got["w"], got["Ls"], got["log_n1"], got["log_n2"]) == (w, ref["Ls"], ref["log_n1"], ref["log_n2"])
            assert abs(got["bound"] - ref["bound"]) <= 1e-9 * ref["bound"]
            assert got["bound"] > prev  # the bound grows with the digit width
            prev = got["bound"]
            if w > proven["w"]:
                assert got["bound"] > 0.49
    for bad in (-1, 31):
        with pytest.raises(hk.HKError):
            hk.fft_plan(0, 64, 3328, w=bad)
