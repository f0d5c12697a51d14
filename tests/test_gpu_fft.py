"""GPU parity of the F3 path (hk_fft_matvec: the paper's decomposition approach with an FP64 FFT,
PAPER.md P:119-170, made exact by Percival's bound -- tests/test_fft_bound.py pins the planner):
bit-exact against the oracle element by element, on every kind, ragged and edge sizes, the
carry-stress recipe, the closed forms with max-magnitude entries (the norms the bound assumes), and
the BASELINE configs (C1 live; C2, C3, C4, C5 via the committed oracle digests).  N1 > 4096 runs the
split column path (first / last column stages from HBM around 4096-point blocks)."""
import hashlib
import json
import os

import numpy as np
import pytest

import hkinputs as gen
import oracle
from oracle import bruteforce as bf

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DIG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "digests")


@pytest.fixture(scope="module")
def hk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1402_5287_b200 as hk
    return hk


def run_fft(hk, kind, am, asg, xm, xsg, P):
    ym, ys = hk.fft_matvec(kind, *hk.to_device(am, asg), *hk.to_device(xm, xsg), P)
    torch.cuda.synchronize()
    return hk.to_host(ym, ys)


def assert_same(got, want, ctx=""):
    gm, gs = got
    wm, ws = want
    bad = np.nonzero((gm != wm).any(axis=1) | (gs != ws))[0]
    assert bad.size == 0, f"{ctx}: {bad.size} rows differ, first {bad[:8]}"


def test_c1_all_kinds(hk):
    for kind in (0, 1, 2):
        am, asg, xm, xsg = gen.make_inputs(kind, 64, 3328, 0)
        assert_same(run_fft(hk, kind, am, asg, xm, xsg, 3328), oracle.matvec(kind, 3328, am, asg, xm, xsg),
                    f"C1 kind={kind}")


@pytest.mark.parametrize("n", [1, 2, 3, 17, 100, 257])
@pytest.mark.parametrize("P", [1, 64, 65, 1000, 5000])
def test_edge_sizes(hk, n, P):
    for kind in (0, 1, 2):
        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=7 * n + P)
        assert_same(run_fft(hk, kind, am, asg, xm, xsg, P), oracle.matvec(kind, P, am, asg, xm, xsg),
                    f"kind={kind} n={n} P={P}")


def test_carry_stress(hk):
    for kind, n in ((1, 200), (2, 256), (2, 77)):
        am, asg, xm, xsg = gen.make_inputs(kind, n, 4000, seed=4, recipe="carry_stress")
        assert_same(run_fft(hk, kind, am, asg, xm, xsg, 4000), oracle.matvec(kind, 4000, am, asg, xm, xsg),
                    f"carry-stress kind={kind} n={n}")


def test_closed_forms_max_magnitude(hk):
    """All entries +(2^P - 1): every digit of the balanced recoding is at its extreme, the largest
    coefficients the bound covers; Y_i = n (2^P - 1)^2 (and the alternating-sign cancellation)."""
    for n, P in ((7, 3328), (64, 16608), (300, 1000), (1000, 2000)):
        Mx = (1 << P) - 1
        for kind in (0, 1, 2):
            am, asg = gen.max_magnitude(gen.a_count(kind, n), P)
            xm, xsg = gen.max_magnitude(n, P)
            assert_same(run_fft(hk, kind, am, asg, xm, xsg, P),
                        bf.from_ints([n * Mx * Mx] * n, gen.n_out_limbs(P)), f"max n={n} P={P} kind={kind}")
        am, asg = gen.max_magnitude(2 * n - 1, P)
        xm, xsg = gen.max_magnitude(n, P, signs=[(-1) ** j for j in range(1, n + 1)])
        assert_same(run_fft(hk, 0, am, asg, xm, xsg, P),
                    bf.from_ints([0 if n % 2 == 0 else -Mx * Mx] * n, gen.n_out_limbs(P)), f"alternating n={n}")


@pytest.mark.parametrize("kind,n,P", [(0, 2100, 1000), (1, 3000, 200), (2, 2049, 500), (2, 8192, 300),
                                      (0, 8200, 64), (1, 5000, 65)])
def test_split_column_path(hk, kind, n, P):
    """N1 = 8192 / 16384 / 32768: f2_top + 4096-row blocks + f2_bottom, every row vs the oracle."""
    assert hk.fft_plan(kind, n, P)["log_n1"] > 12
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=n + P)
    assert_same(run_fft(hk, kind, am, asg, xm, xsg, P), oracle.matvec(kind, P, am, asg, xm, xsg),
                f"split kind={kind} n={n} P={P}")


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5T", "C5C"])
def test_config_digest(hk, name):
    if not os.path.exists(os.path.join(DIG, f"{name}.json")):
        pytest.skip(f"no committed oracle digest for {name} yet")
    meta = json.load(open(os.path.join(DIG, f"{name}.json")))
    c = gen.CONFIGS[name]
    am, asg, xm, xsg = gen.config_inputs(name)
    gm, gs = run_fft(hk, c["kind"], am, asg, xm, xsg, c["P"])
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(gm).tobytes())
    h.update(np.ascontiguousarray(gs).tobytes())
    if meta.get("y_sha256"):
        assert h.hexdigest() == meta["y_sha256"], f"{name}: FFT-path y differs from the oracle digest"
        return
    # C4: the oracle run was split between hosts and kept row digests only (scripts/oracle_digests.py)
    want = open(os.path.join(DIG, f"{name}.rows")).read().split()
    assert len(want) == gm.shape[0] and meta.get("rows_missing", 0) == 0
    bad = [i for i, w in enumerate(want)
           if hashlib.sha256(gm[i].tobytes() + gs[i:i + 1].tobytes()).hexdigest()[:16] != w]
    assert not bad, f"{name}: FFT-path y differs from the oracle's in {len(bad)} rows, first {bad[:8]}"


def test_rejects_bits_above_P(hk):
    P = 300
    am, asg, xm, xsg = gen.make_inputs(0, 20, P, seed=3)
    am = am.copy()
    am[2, -1] |= np.uint64(1) << np.uint64(63)
    with pytest.raises(hk.HKError):
        run_fft(hk, 0, am, asg, xm, xsg, P)


def test_workspace_reuse(hk):
    n, P = 150, 3000
    ws = hk.FftWorkspace(0, n, P)
    for seed in (1, 2):
        am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=seed)
        a, sa = hk.to_device(am, asg)
        x, sx = hk.to_device(xm, xsg)
        got = hk.to_host(*hk.fft_matvec(0, a, sa, x, sx, P, ws=ws))
        assert_same(got, oracle.matvec(0, P, am, asg, xm, xsg), f"reuse seed={seed}")


def test_forced_width_study_path(hk):
    """F3 accuracy study entry points (hk_fft_matvec_w): at the proven width the forced-w path is the
    product path (same y, the oracle's) and its measured max |v - rint(v)| stays under the Percival
    bound; at wider widths, whenever every residual is below 1/2 the rounded coefficients are the
    exact integers, so y must still equal the oracle's (a residual >= 1/2 is allowed to break it)."""
    kind, n, P = 0, 96, 3328
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=11)
    want = oracle.matvec(kind, P, am, asg, xm, xsg)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    proven = hk.fft_plan(kind, n, P)
    for w in (proven["w"], proven["w"] + 2, proven["w"] + 4, proven["w"] + 8):
        info = hk.fft_plan(kind, n, P, w=w)
        res = torch.zeros(1, dtype=torch.float64, device=a.device)
        ym, ys = hk.fft_matvec(kind, a, sa, x, sx, P, w=w, residual=res)
        torch.cuda.synchronize()
        r = float(res.item())
        got = hk.to_host(ym, ys)
        if w == proven["w"]:
            assert 0.0 < r <= info["bound"] < 0.5, (w, r, info["bound"])
            assert_same(got, want, f"proven w={w}")
        elif r < 0.5:
            assert_same(got, want, f"w={w} residual {r}")
    # a workspace initialised for one width is refused by a call with another
    ws = hk.FftWorkspace(kind, n, P, w=proven["w"] + 2)
    with pytest.raises(ValueError):
        hk.fft_matvec(kind, a, sa, x, sx, P, ws=ws)
