"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/hk.h declares,
and its host-side logic (planner capacity proof, argument validation) behaves.  No GPU compute."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1402_5287_b200 as hk
from tests import fingerprint as fp
import hkinputs as gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRIMES = [2147352577, 2146959361, 2146041857, 2144468993, 2142502913]


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(hk.library_path())
    names = declared_symbols()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(hk.EXPORTED)


def test_limbs():
    assert hk.limbs(1) == 1 and hk.limbs(64) == 1 and hk.limbs(65) == 2
    assert hk.limbs(33216) == 519 and hk.out_limbs(33216) == 1039
    assert hk.limbs(0) == -1


def test_status_strings():
    for c in (0, -1, -2, -3, -4, -5):
        assert hk.status_string(c).startswith("HK_")


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5T", "C5C"])
def test_plan_capacity_proof(name):
    """2 n Ls (2^w-1)^2 < p1..p5 (symmetric CRT recovers every coefficient exactly), the
    slice transform holds the linear convolution (N2 >= 2Ls-1) and the matrix-index transform
    holds the needed convolution (N1 >= 2n-1, or N1 = n for a power-of-two circulant)."""
    c = gen.CONFIGS[name]
    pl = hk.plan(c["kind"], c["n"], c["P"])
    M = math.prod(PRIMES)
    assert 2 * c["n"] * pl["Ls"] * ((1 << pl["w"]) - 1) ** 2 < M
    assert pl["Ls"] == -(-c["P"] // pl["w"]) and pl["w"] <= 65
    assert (1 << pl["log_n2"]) >= 2 * pl["Ls"] - 1
    if pl["cyclic"]:
        assert (1 << pl["log_n1"]) == c["n"]
    else:
        assert (1 << pl["log_n1"]) >= 2 * c["n"] - 1
    assert pl["margin_bits"] > 0


def test_plan_c3_matches_design():
    pl = hk.plan(0, 8000, 33216)
    assert (pl["w"], pl["Ls"], pl["log_n2"], pl["log_n1"]) == (65, 512, 10, 14)
    assert 1.9 < pl["margin_bits"] < 2.2
    pl4 = hk.plan(0, 16384, 33216)
    assert pl4["log_n1"] == 15 and 0.9 < pl4["margin_bits"] < 1.1


def test_plan_limits_and_errors():
    with pytest.raises(hk.HKError) as e:
        hk.plan(0, 16385, 33216)  # N1 > 32768
    assert e.value.code == hk.HK_EUNSUPPORTED
    with pytest.raises(hk.HKError) as e:
        hk.plan(0, 0, 64)
    assert e.value.code == hk.HK_EINVAL
    with pytest.raises(hk.HKError):
        hk.plan(0, 4, 0)
    with pytest.raises(hk.HKError):
        hk.plan(3, 4, 64)
    # rectangular Hankel window: N1 >= m + n - 1
    pl = hk.plan(0, 8000, 33216, m=1000)
    assert (1 << pl["log_n1"]) >= 8999 and pl["a_count"] == 8999


def test_workspace_size_monotone():
    a = hk.workspace_size(0, 1000, 33216)
    b = hk.workspace_size(0, 2000, 33216)
    s = hk.workspace_size(0, 1000, 33216, flags=hk.WS_STAGING)
    pr = hk.workspace_size(0, 1000, 33216, flags=hk.WS_PREPARED)
    assert 0 < a < b and s > a and pr > a
    with pytest.raises(hk.HKError):  # staging and prepared are mutually exclusive
        hk.workspace_size(0, 1000, 33216, flags=hk.WS_STAGING | hk.WS_PREPARED)


def test_null_pointer_arguments_rejected_synchronously():
    rc = hk._lib.hk_hankel_matvec(4, 64, None, None, None, None, None, None, None, 0, None)
    assert rc == hk.HK_EINVAL
    rc = hk._lib.hk_schoolbook_matvec(0, 4, 4, 64, None, None, None, None, None, None, None)
    assert rc == hk.HK_EINVAL


def test_fingerprint_helper_against_oracle():
    """The test-side fingerprint reproduces the oracle's rows mod q (pins the helper)."""
    import oracle
    for kind in (0, 1, 2):
        am, asg, xm, xsg = gen.make_inputs(kind, 13, 700, seed=kind + 50)
        ym, ys = oracle.matvec(kind, 700, am, asg, xm, xsg, threads=2)
        fp.check(kind, am, asg, xm, xsg, ym, ys)
    am, asg, xm, xsg = gen.make_inputs(0, 9, 300, seed=77, m=4)
    ym, ys = oracle.matvec(0, 300, am, asg, xm, xsg, m=4, threads=2)
    fp.check(0, am, asg, xm, xsg, ym, ys, m=4)
