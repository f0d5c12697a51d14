"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bit-exact on every output limb and sign (all inputs are integers; reading R10 makes
the byte image unique).  Full-oracle cases span several tiles and ragged tails; the BASELINE
configs at full size are checked on sampled rows with the oracle plus modular fingerprints of
every row (tests/fingerprint.py), in the launch configuration bench.py times."""
import numpy as np
import pytest

import hkinputs as gen
import oracle
from oracle import bruteforce as bf
from tests import fingerprint as fp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1402_5287_b200 as hk
    return hk


def run_gpu(hk, kind, a_mag, a_sign, x_mag, x_sign, P, m=None, ws=None):
    am, asg = hk.to_device(a_mag, a_sign)
    xm, xsg = hk.to_device(x_mag, x_sign)
    ym, ys = hk.matvec(kind, am, asg, xm, xsg, P, m=m, ws=ws)
    torch.cuda.synchronize()
    return hk.to_host(ym, ys)


def assert_same(got, want, ctx=""):
    gm, gs = got
    wm, ws = want
    bad = np.nonzero((gm != wm).any(axis=1) | (gs != ws))[0]
    assert bad.size == 0, f"{ctx}: {bad.size} rows differ, first {bad[:8]}"


def full_case(hk, kind, n, P, seed, recipe="uniform", m=None):
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed, recipe, m=m)
    got = run_gpu(hk, kind, am, asg, xm, xsg, P, m=m)
    want = oracle.matvec(kind, P, am, asg, xm, xsg, m=m)
    assert_same(got, want, f"kind={kind} n={n} P={P} m={m}")


# ---------------------------------------------------------------------------------------------
def test_c1_all_kinds(hk):
    for kind in (0, 1, 2):
        full_case(hk, kind, 64, 3328, 0)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 33, 100, 257])
@pytest.mark.parametrize("P", [1, 64, 65, 127, 1000])
def test_small_edge_sizes(hk, n, P):
    for kind in (0, 1, 2):
        full_case(hk, kind, n, P, seed=n * 1000 + P)


@pytest.mark.parametrize("n,P", [(300, 5000), (129, 33216), (1000, 700), (64, 16608)])
def test_medium_full_oracle(hk, n, P):
    for kind in (0, 1, 2):
        full_case(hk, kind, n, P, seed=n + P)


@pytest.mark.parametrize("n", [64, 128, 512])
def test_cyclic_circulant_power_of_two(hk, n):
    assert hk.plan(2, n, 2000)["cyclic"] == 1
    full_case(hk, 2, n, 2000, seed=n)


def test_carry_stress_small(hk):
    for kind in (1, 2):
        full_case(hk, kind, 200, 4000, seed=4, recipe="carry_stress")


def test_closed_forms(hk):
    """max magnitude everywhere (largest output) and alternating signs (exact cancellation)."""
    for n, P in [(7, 3328), (64, 16608), (300, 1000)]:
        for kind in (0, 1, 2):
            am, asg = gen.max_magnitude(gen.a_count(kind, n), P)
            xm, xsg = gen.max_magnitude(n, P)
            got = run_gpu(hk, kind, am, asg, xm, xsg, P)
            Mx = (1 << P) - 1
            want = bf.from_ints([n * Mx * Mx] * n, gen.n_out_limbs(P))
            assert_same(got, want, f"max n={n} P={P} kind={kind}")
        am, asg = gen.max_magnitude(2 * n - 1, P)
        xm, xsg = gen.max_magnitude(n, P, signs=[(-1) ** j for j in range(1, n + 1)])
        got = run_gpu(hk, 0, am, asg, xm, xsg, P)
        Mx = (1 << P) - 1
        want = bf.from_ints([0 if n % 2 == 0 else -Mx * Mx] * n, gen.n_out_limbs(P))
        assert_same(got, want, f"alternating n={n}")


def test_zero_inputs(hk):
    am, asg = gen.zeros(2 * 50 - 1, 3000)
    xm, xsg = gen.uniform(1, 1, 50, 3000)
    gm, gs = run_gpu(hk, 0, am, asg, xm, xsg, 3000)
    assert not gm.any() and not gs.any()


def test_rect_windows(hk):
    """Row-block shards: m x n windows of a Hankel product."""
    for (m, n) in [(1, 200), (37, 100), (250, 250), (100, 37)]:
        full_case(hk, 0, n, 3000, seed=m + n, m=m)


@pytest.mark.parametrize("kind,n", [(0, 200), (1, 203), (2, 128), (2, 77), (0, 5), (1, 1)])
def test_host_buffer_path(hk, kind, n):
    """hk_matvec_host: chunked H2D / K1, K2, chunked K3 / D2H pipeline."""
    am, asg, xm, xsg = gen.make_inputs(kind, n, 5000, seed=3 + n)
    ym, ys = hk.matvec_host(kind, am, asg, xm, xsg, 5000)
    assert_same((ym, ys), oracle.matvec(kind, 5000, am, asg, xm, xsg), "host path")


@pytest.mark.parametrize("kind,n,P", [(0, 200, 5000), (1, 77, 3328), (2, 128, 1000), (2, 33, 700)])
def test_host_pipeline_async(hk, kind, n, P):
    """hk_matvec_host_async through HostPipeline: 7 different problems over 3 lanes in flight."""
    import torch
    pipe = hk.HostPipeline(kind, n, P, depth=3)
    Ly = hk.out_limbs(P)
    cases, outs = [], []
    for t in range(7):
        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=100 + t,
                                           recipe="carry_stress" if t % 2 else "uniform")
        host = [torch.from_numpy(v.view(np.int64) if v.dtype == np.uint64 else v).pin_memory()
                for v in (am, asg, xm, xsg)]
        out = (torch.empty((n, Ly), dtype=torch.int64).pin_memory(),
               torch.empty((n,), dtype=torch.int8).pin_memory())
        pipe.submit(*host, out)
        cases.append((am, asg, xm, xsg, host))
        outs.append(out)
    pipe.drain()
    for (am, asg, xm, xsg, _), (ym, ys) in zip(cases, outs):
        got = (ym.numpy().view(np.uint64), ys.numpy())
        assert_same(got, oracle.matvec(kind, P, am, asg, xm, xsg), "host pipeline")


def test_host_pipeline_reports_data_error(hk):
    import torch
    n, P = 40, 200
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=5)
    xm = xm.copy()
    xm[3, -1] |= np.uint64(1) << np.uint64(63)  # bit >= P set
    pipe = hk.HostPipeline(0, n, P, depth=2)
    host = [torch.from_numpy(v.view(np.int64) if v.dtype == np.uint64 else v).pin_memory()
            for v in (am, asg, xm, xsg)]
    out = (torch.empty((n, hk.out_limbs(P)), dtype=torch.int64).pin_memory(),
           torch.empty((n,), dtype=torch.int8).pin_memory())
    pipe.submit(*host, out)
    with pytest.raises(hk.HKError):
        pipe.drain()


def test_workspace_reuse_and_determinism(hk):
    am, asg, xm, xsg = gen.make_inputs(0, 500, 8000, seed=12)
    ws = hk.Workspace(0, 500, 8000)
    r1 = run_gpu(hk, 0, am, asg, xm, xsg, 8000, ws=ws)
    r2 = run_gpu(hk, 0, am, asg, xm, xsg, 8000, ws=ws)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])
    fp.check(0, am, asg, xm, xsg, *r1)


# ---------------------------------------------------------------------------------------------
# data validation (fault injection)
def _expect_status(hk, kind, am, asg, xm, xsg, P, code):
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ws = hk.Workspace(kind, xm.shape[0], P)
    hk.matvec(kind, a, sa, x, sx, P, ws=ws, check=False)
    assert ws.status() == code


def test_rejects_bits_above_P(hk):
    P = 100
    am, asg, xm, xsg = gen.make_inputs(0, 20, P, seed=1)
    am[5, 1] |= np.uint64(1 << 40)  # bit 104 >= P
    _expect_status(hk, 0, am, asg, xm, xsg, P, hk.HK_ERANGE)


def test_rejects_sign_magnitude_mismatch(hk):
    P = 200
    am, asg, xm, xsg = gen.make_inputs(0, 20, P, seed=2)
    xsg = xsg.copy(); xm = xm.copy()
    xm[3] = 0; xsg[3] = 1  # zero magnitude with sign +1
    _expect_status(hk, 0, am, asg, xm, xsg, P, hk.HK_ERANGE)
    am, asg, xm, xsg = gen.make_inputs(0, 20, P, seed=2)
    asg = asg.copy(); asg[7] = 2
    _expect_status(hk, 0, am, asg, xm, xsg, P, hk.HK_ERANGE)
    am, asg, xm, xsg = gen.make_inputs(0, 20, P, seed=2)
    asg = asg.copy(); asg[0] = 0  # non-zero magnitude with sign 0
    _expect_status(hk, 0, am, asg, xm, xsg, P, hk.HK_ERANGE)


def test_uninitialised_workspace(hk):
    P = 128
    am, asg, xm, xsg = gen.make_inputs(0, 10, P, seed=3)
    ws = hk.Workspace(0, 11, P)  # initialised for n = 11, used for n = 10 -> rejected by binding
    with pytest.raises(ValueError):
        hk.matvec(0, *hk.to_device(am, asg), *hk.to_device(xm, xsg), P, ws=ws)
    # a zeroed buffer passed through the raw ABI -> device-side EINVAL
    nbytes = hk.workspace_size(0, 10, P)
    buf = torch.zeros(nbytes + 256, dtype=torch.uint8, device="cuda")
    ptr = (buf.data_ptr() + 255) & ~255
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    y = torch.empty((10, gen.n_out_limbs(P)), dtype=torch.int64, device="cuda")
    ysg = torch.empty(10, dtype=torch.int8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rc = hk._lib.hk_hankel_matvec(10, P, a.data_ptr(), sa.data_ptr(), x.data_ptr(), sx.data_ptr(),
                                  y.data_ptr(), ysg.data_ptr(), ptr, nbytes, s)
    assert rc == hk.HK_OK
    import ctypes
    v = ctypes.c_int32()
    assert hk._lib.hk_workspace_status(ptr, s, ctypes.byref(v)) == 0
    assert v.value == hk.HK_EINVAL


def test_undersized_workspace_and_overlap(hk):
    P = 128
    am, asg, xm, xsg = gen.make_inputs(0, 10, P, seed=3)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ws = hk.Workspace(0, 10, P)
    s = torch.cuda.current_stream().cuda_stream
    y = torch.empty((10, gen.n_out_limbs(P)), dtype=torch.int64, device="cuda")
    ysg = torch.empty(10, dtype=torch.int8, device="cuda")
    rc = hk._lib.hk_hankel_matvec(10, P, a.data_ptr(), sa.data_ptr(), x.data_ptr(), sx.data_ptr(),
                                  y.data_ptr(), ysg.data_ptr(), ws.ptr, ws.nbytes - 1024, s)
    assert rc == hk.HK_ENOMEM
    rc = hk._lib.hk_hankel_matvec(10, P, a.data_ptr(), sa.data_ptr(), x.data_ptr(), sx.data_ptr(),
                                  a.data_ptr(), ysg.data_ptr(), ws.ptr, ws.nbytes, s)
    assert rc == hk.HK_EINVAL


# ---------------------------------------------------------------------------------------------
# BASELINE configs at full size (sampled rows + fingerprints of every row)
SAMPLE_ROWS = 12


def _sampled(hk, name, rows_extra=()):
    c = gen.CONFIGS[name]
    kind, n, P = c["kind"], c["n"], c["P"]
    am, asg, xm, xsg = gen.config_inputs(name)
    gm, gs = run_gpu(hk, kind, am, asg, xm, xsg, P)
    fp.check(kind, am, asg, xm, xsg, gm, gs)
    rng = np.random.default_rng(123)
    rows = np.unique(np.concatenate([np.array([0, 1, n // 2, n - 2, n - 1], dtype=np.int64),
                                     rng.integers(0, n, SAMPLE_ROWS).astype(np.int64),
                                     np.asarray(rows_extra, dtype=np.int64)]))
    wm, ws_ = oracle.matvec(kind, P, am, asg, xm, xsg, rows=rows)
    assert_same((gm[rows], gs[rows]), (wm, ws_), f"{name} sampled rows")


def test_c2_full_oracle(hk):
    """BASELINE configs[1] in full: every row against a live oracle run (and the fingerprints)."""
    c = gen.CONFIGS["C2"]
    am, asg, xm, xsg = gen.config_inputs("C2")
    got = run_gpu(hk, 0, am, asg, xm, xsg, c["P"])
    fp.check(0, am, asg, xm, xsg, *got)
    assert_same(got, oracle.matvec(0, c["P"], am, asg, xm, xsg), "C2 all rows")


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("P", [64, 200])
def test_n1_2p14_all_rows(hk, kind, P):
    """n = 8000: the N1 = 2^14 column kernel C3 runs (256-thread K2, 2 CTAs/SM, shared-memory
    twiddles), at a small P so the oracle finishes every row in seconds."""
    full_case(hk, kind, 8000, P, seed=8000 + P + kind)


def test_n1_2p14_all_rows_n2_128(hk):
    full_case(hk, 0, 8000, 2100, seed=82100)  # Ls = 33, N2 = 128


@pytest.mark.parametrize("name", ["C3", "C4", "C5T", "C5C"])
def test_config_sampled(hk, name):
    _sampled(hk, name)


# ---------------------------------------------------------------------------------------------
# companion A6: schoolbook kernel
@pytest.mark.parametrize("n,P", [(1, 64), (1, 1), (2, 32), (5, 65), (7, 33), (64, 3328), (100, 1000),
                                 (33, 16608), (300, 200), (257, 3328), (5, 40000), (3, 33216)])
def test_schoolbook_parity(hk, n, P):
    for kind in (0, 1, 2):
        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=n + 7)
        a, sa = hk.to_device(am, asg)
        x, sx = hk.to_device(xm, xsg)
        ym, ys = hk.schoolbook_matvec(kind, a, sa, x, sx, P)
        torch.cuda.synchronize()
        assert_same(hk.to_host(ym, ys), oracle.matvec(kind, P, am, asg, xm, xsg),
                    f"schoolbook kind={kind} n={n} P={P}")


def test_schoolbook_carry_stress_and_rect(hk):
    """Carry-stress mantissas (long runs of ones / zeros, signs mixed) for all kinds, and the
    rectangular Hankel window (m < n rows) that the row-block plan uses."""
    for kind, n, P in ((0, 96, 3328), (1, 64, 1000), (2, 48, 16608)):
        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=3, recipe="carry_stress")
        a, sa = hk.to_device(am, asg)
        x, sx = hk.to_device(xm, xsg)
        ym, ys = hk.schoolbook_matvec(kind, a, sa, x, sx, P)
        torch.cuda.synchronize()
        assert_same(hk.to_host(ym, ys), oracle.matvec(kind, P, am, asg, xm, xsg), f"stress {kind}")
    n, m, P = 40, 9, 2000
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=5)
    am, asg = am[: m + n - 1], asg[: m + n - 1]
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ym, ys = hk.schoolbook_matvec(0, a, sa, x, sx, P, m=m)
    torch.cuda.synchronize()
    want = oracle.matvec(0, P, am, asg, xm, xsg, m=m)
    assert_same(hk.to_host(ym, ys), want, "rect")


def test_schoolbook_max_magnitude(hk):
    """Closed form: every entry +(2^P - 1) gives y_i = n (2^P - 1)^2 (the largest output)."""
    n, P = 37, 1000
    L = (P + 63) // 64
    full = np.zeros(L, dtype=np.uint64)
    for l in range(L):
        bits = min(64, P - 64 * l)
        full[l] = np.uint64((1 << bits) - 1)
    am = np.tile(full, (2 * n - 1, 1)); asg = np.ones(2 * n - 1, dtype=np.int8)
    xm = np.tile(full, (n, 1)); xsg = np.ones(n, dtype=np.int8)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ym, ys = hk.to_host(*hk.schoolbook_matvec(0, a, sa, x, sx, P))
    want = n * ((1 << P) - 1) ** 2
    for i in range(n):
        got = sum(int(ym[i, l]) << (64 * l) for l in range(ym.shape[1]))
        assert got == want and ys[i] == 1


# ---------------------------------------------------------------------------------------------
# companion A5: Algorithm 1 level by level
@pytest.mark.parametrize("n,P,cutoff", [(1, 64, 2), (2, 64, 2), (3, 100, 2), (5, 65, 2),
                                        (17, 1000, 2), (64, 3328, 2), (64, 3328, 8),
                                        (100, 2000, 4), (129, 700, 8), (33, 16608, 2),
                                        (257, 200, 3)])
def test_karatsuba_parity(hk, n, P, cutoff):
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=n + cutoff)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ym, ys = hk.karatsuba_matvec(a, sa, x, sx, P, cutoff=cutoff)
    torch.cuda.synchronize()
    assert_same(hk.to_host(ym, ys), oracle.matvec(0, P, am, asg, xm, xsg),
                f"karatsuba n={n} P={P} cutoff={cutoff}")


def test_karatsuba_carry_stress_and_c2_rows(hk):
    am, asg, xm, xsg = gen.make_inputs(0, 64, 16608, seed=4, recipe="carry_stress")
    got = hk.to_host(*hk.karatsuba_matvec(*hk.to_device(am, asg), *hk.to_device(xm, xsg), 16608,
                                          cutoff=2))
    assert_same(got, oracle.matvec(0, 16608, am, asg, xm, xsg), "karatsuba carry-stress")
    am, asg, xm, xsg = gen.config_inputs("C2")
    got = hk.to_host(*hk.karatsuba_matvec(*hk.to_device(am, asg), *hk.to_device(xm, xsg), 33216,
                                          cutoff=8))
    fp.check(0, am, asg, xm, xsg, *got)
    rows = np.array([0, 1, 511, 1022, 1023], dtype=np.int64)
    wm, ws_ = oracle.matvec(0, 33216, am, asg, xm, xsg, rows=rows)
    assert_same((got[0][rows], got[1][rows]), (wm, ws_), "karatsuba C2 rows")


# ---------------------------------------------------------------------------------------------
# F1: fixed-A repeated products (prepared transform of a)
@pytest.mark.parametrize("kind,n,P", [(0, 64, 3328), (1, 100, 2000), (2, 128, 1000), (2, 77, 700),
                                      (0, 1, 64), (0, 1000, 33216)])
def test_prepared_matrix_many_vectors(hk, kind, n, P):
    am, asg, _, _ = gen.make_inputs(kind, n, P, seed=31 + n)
    A = hk.PreparedMatrix(kind, *hk.to_device(am, asg), P, n)
    for v in range(3):
        xm, xsg = gen.uniform(100 + v, 1, n, P)
        got = hk.to_host(*A.matvec(*hk.to_device(xm, xsg)))
        if n <= 200:
            want = oracle.matvec(kind, P, am, asg, xm, xsg)
            assert_same(got, want, f"prepared kind={kind} n={n} v={v}")
        else:
            fp.check(kind, am, asg, xm, xsg, *got)


@pytest.mark.parametrize("kind,n,P,lanes", [(0, 64, 3328, 2), (1, 100, 2000, 3), (2, 77, 700, 2),
                                            (0, 33, 65, 4)])
def test_prepared_matrix_batch_lanes(hk, kind, n, P, lanes):
    """F1 multi-vector batching: vectors spread over lanes (streams with their own prepared copy)."""
    am, asg, _, _ = gen.make_inputs(kind, n, P, seed=41 + n)
    A = hk.PreparedMatrix(kind, *hk.to_device(am, asg), P, n, lanes=lanes)
    xs_host = [gen.uniform(200 + v, 1, n, P) for v in range(2 * lanes + 1)]
    ys = A.matvec_batch([hk.to_device(xm, xsg) for xm, xsg in xs_host])
    assert len(ys) == len(xs_host)
    for v, ((xm, xsg), y) in enumerate(zip(xs_host, ys)):
        want = oracle.matvec(kind, P, am, asg, xm, xsg)
        assert_same(hk.to_host(*y), want, f"batch kind={kind} n={n} lanes={lanes} v={v}")


def test_prepared_requires_prepare(hk):
    P, n = 128, 10
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=3)
    ws = hk.Workspace(0, n, P, flags=hk.WS_PREPARED)  # initialised, never prepared
    x, sx = hk.to_device(xm, xsg)
    y = torch.empty((n, gen.n_out_limbs(P)), dtype=torch.int64, device="cuda")
    ysg = torch.empty(n, dtype=torch.int8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rc = hk._lib.hk_matvec_prepared(0, n, n, P, x.data_ptr(), sx.data_ptr(), y.data_ptr(),
                                    ysg.data_ptr(), ws.ptr, ws.nbytes, s)
    assert rc == hk.HK_OK and ws.status() == hk.HK_EINVAL


# ---------------------------------------------------------------------------------------------
# F4: y rounded back to the input format (hk_matvec_rounded) vs the oracle's exact y rounded
# by oracle/rounding.py (round half to even, pinned to round(Fraction) in test_oracle_pins.py)
def run_gpu_rounded(hk, kind, am, asg, xm, xsg, P, m=None):
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ym, ys = hk.matvec(kind, a, sa, x, sx, P, m=m, rounded=True)
    torch.cuda.synchronize()
    return hk.to_host(ym, ys)


@pytest.mark.parametrize("kind,n,P,recipe", [
    (0, 64, 3328, "uniform"), (1, 33, 1000, "uniform"), (2, 128, 700, "uniform"),
    (2, 77, 2000, "carry_stress"), (0, 300, 5000, "carry_stress"), (0, 1, 64, "uniform"),
    (1, 17, 65, "carry_stress"), (0, 129, 33216, "uniform")])
def test_rounded_output(hk, kind, n, P, recipe):
    from oracle import rounding as rd
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=60 + n, recipe=recipe)
    got = run_gpu_rounded(hk, kind, am, asg, xm, xsg, P)
    want = rd.round_rows(*oracle.matvec(kind, P, am, asg, xm, xsg), P)
    assert_same(got, want, "rounded")


@pytest.mark.parametrize("P", [1, 63, 64, 65, 130])
def test_rounded_output_exact_ties(hk, P):
    """Hankel rows whose exact value is k + 1/2 in units of 2^-P (ties go to the even k), plus
    exact integers and a canonical zero."""
    from oracle import rounding as rd
    n, L = 4, (P + 63) // 64
    half = 1 << (P - 1)
    a_vals = [-1, 0, 0, 1, 1, 1, 0]          # a_1 .. a_7 (|a| < 2^P for every P >= 1)
    x_vals = [half, half, half, 0]           # Y_i = (a_i + a_i+1 + a_i+2) 2^(P-1)
    to = lambda vals: (np.array([rd.int_to_limbs(abs(v), L) for v in vals], dtype=np.uint64),
                       np.array([(v > 0) - (v < 0) for v in vals], dtype=np.int8))
    am, asg = to(a_vals)
    xm, xsg = to(x_vals)
    got = run_gpu_rounded(hk, 0, am, asg, xm, xsg, P)
    want = rd.round_rows(*oracle.matvec(0, P, am, asg, xm, xsg), P)
    assert_same(got, want, "rounded ties")
    # -1/2 -> 0 (canonical zero), 1/2 -> 0, exactly 1, 3/2 -> 2
    assert [int(v) for v in got[0][:, 0]] == [0, 0, 1, 2] and list(got[1]) == [0, 0, 1, 1]


def test_split_k2_large_n1(hk):
    """N1 = 2^15 (n > 8192) runs K2 as prepare + prepared launches through the workspace's AT
    region: bit-exact (all rows, small P), a prepared matrix in the same workspace serves
    vectors, and a cold call on that workspace invalidates it (AT overwritten)."""
    n, P = 8200, 64
    assert hk.plan(0, n, P)["log_n1"] == 15
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=77)
    got = run_gpu(hk, 0, am, asg, xm, xsg, P)
    assert_same(got, oracle.matvec(0, P, am, asg, xm, xsg), "split K2")
    A = hk.PreparedMatrix(0, *hk.to_device(am, asg), P, n)
    x2m, x2s = gen.uniform(9, 1, n, P)
    assert_same(hk.to_host(*A.matvec(*hk.to_device(x2m, x2s))),
                oracle.matvec(0, P, am, asg, x2m, x2s), "split K2 prepared")
    hk.matvec(0, *hk.to_device(am, asg), *hk.to_device(xm, xsg), P, ws=A.ws)  # cold call, same ws
    with pytest.raises(hk.HKError):
        A.matvec(*hk.to_device(x2m, x2s))


@pytest.mark.parametrize("kind,n,P", [(0, 33, 33281), (1, 20, 40000), (2, 64, 66560), (0, 7, 66000)])
def test_large_P_slice_transform_2048(hk, kind, n, P):
    """P > 33,280 bits: slice transform N2 = 2048 (K1 / K3 instances with LOGN2 = 11, K3 tiles of
    2 rows), up to the planner's limit P = 66,560 (Ls = 1024)."""
    assert hk.plan(kind, n, P)["log_n2"] == 11
    full_case(hk, kind, n, P, seed=P % 97)
    full_case(hk, kind, n, P, seed=P % 89, recipe="carry_stress")


def test_planner_limit(hk):
    with pytest.raises(hk.HKError):
        hk.plan(0, 10, 66561)


def test_misaligned_magnitudes_rejected(hk):
    """Magnitude arrays must be 16-byte aligned (16-byte / TMA bulk staging): HK_EINVAL, not a fault."""
    n, P = 5, 64
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=1)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    big = torch.empty((2 * n, 1), dtype=torch.int64, device="cuda")
    a_off = big[1: 2 * n]  # 8-byte offset view
    a_off.copy_(a)
    ws = hk.Workspace(0, n, P)
    y = torch.empty((n, hk.out_limbs(P)), dtype=torch.int64, device="cuda")
    ys = torch.empty(n, dtype=torch.int8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rc = hk._lib.hk_hankel_matvec(n, P, a_off.data_ptr(), sa.data_ptr(), x.data_ptr(), sx.data_ptr(),
                                  y.data_ptr(), ys.data_ptr(), ws.ptr, ws.nbytes, s)
    assert rc == hk.HK_EINVAL


# ---------------------------------------------------------------------------------------------
# round-2 hazards: data status across prepared / batched calls, shard alignment
def test_prepare_with_rejected_a_poisons_later_calls(hk):
    """hk_prepare_a on an a with a bit >= P: a_ready stays 0, so every later prepared matvec
    reports an error instead of computing with the rejected matrix."""
    n, P = 30, 300
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=9)
    am = am.copy()
    am[4, -1] |= np.uint64(1) << np.uint64(63)
    A = hk.PreparedMatrix(0, *hk.to_device(am, asg), P, n, check=False)
    assert A.ws.status() == hk.HK_ERANGE
    for _ in range(2):
        with pytest.raises(hk.HKError):
            A.matvec(*hk.to_device(xm, xsg))


def test_matvec_batch_reports_each_vectors_status(hk):
    """More vectors than lanes: a rejected x in an early round is reported even though later
    calls on the same lane reset the lane's status word."""
    n, P, lanes = 40, 500, 2
    am, asg, _, _ = gen.make_inputs(0, n, P, seed=10)
    A = hk.PreparedMatrix(0, *hk.to_device(am, asg), P, n, lanes=lanes)
    xs = [gen.uniform(300 + v, 1, n, P) for v in range(2 * lanes + 1)]
    bad = 1
    xm_bad = xs[bad][0].copy()
    xm_bad[0, -1] |= np.uint64(1) << np.uint64(62)
    xs[bad] = (xm_bad, xs[bad][1])
    with pytest.raises(hk.HKError, match=f"vector {bad}"):
        A.matvec_batch([hk.to_device(xm, xsg) for xm, xsg in xs])
    ys = A.matvec_batch([hk.to_device(xm, xsg) for xm, xsg in xs[2:]])  # the others are fine
    for (xm, xsg), y in zip(xs[2:], ys):
        assert_same(hk.to_host(*y), oracle.matvec(0, P, am, asg, xm, xsg), "batch after error")


def test_rowblock_window_alignment(hk):
    """A row-block window starting r0 L 8 bytes into a_mag is only 8-byte aligned when r0 L is odd;
    the C ABI rejects it (HK_EINVAL) and dist.ShardedHankel therefore uses its own copy."""
    from paper_1402_5287_b200 import dist as hkdist
    n, P = 50, 3 * 64 - 5  # L = 3 (odd)
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=11)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    r0, nr = 7, 20  # r0 L = 21: odd
    wm, wsg = hkdist.window(a, sa, r0, nr, n)
    with pytest.raises(hk.HKError):
        hk.hankel_rect_matvec(wm, wsg, x, sx, P, nr)
    got = hk.hankel_rect_matvec(wm.clone(), wsg.clone(), x, sx, P, nr)
    want = oracle.matvec(0, P, am, asg, xm, xsg, rows=np.arange(r0, r0 + nr))
    assert_same(hk.to_host(*got), want, "aligned window copy")


def test_circulant_w64_plan(hk):
    """Circulant n = 32768 (cyclic N1 = 2^15), P = 33,216: the capacity bound rules out w = 65, so
    the planner takes w = 64, N2 = 2048 (K3 with 2-row tiles).  Fingerprints of every row and
    three rows against the oracle."""
    n, P = 32768, 33216
    pl = hk.plan(2, n, P)
    assert pl["w"] == 64 and pl["log_n2"] == 11 and pl["cyclic"] == 1
    am, asg, xm, xsg = gen.make_inputs(2, n, P, seed=64)
    gm, gs = run_gpu(hk, 2, am, asg, xm, xsg, P)
    fp.check(2, am, asg, xm, xsg, gm, gs)
    rows = np.array([0, 12345, n - 1])
    wm, ws_ = oracle.matvec(2, P, am, asg, xm, xsg, rows=rows)
    assert_same((gm[rows], gs[rows]), (wm, ws_), "w=64 circulant rows")


# ---------------------------------------------------------------------------------------------
# F1 kernel-level batch (hk_matvec_prepared_batch): one launch per kernel for several vectors
@pytest.mark.parametrize("kind,n,P,batch", [(0, 300, 5000, 3), (1, 77, 3328, 2), (2, 128, 1000, 4),
                                            (2, 77, 700, 3), (0, 8200, 64, 2)])
def test_prepared_batch_kernel_level(hk, kind, n, P, batch):
    am, asg, _, _ = gen.make_inputs(kind, n, P, seed=61 + n)
    A = hk.PreparedMatrix(kind, *hk.to_device(am, asg), P, n, batch=batch)
    xs_host = [gen.uniform(400 + v, 1, n, P) for v in range(2 * batch + 1)]
    ys = A.matvec_batch([hk.to_device(xm, xsg) for xm, xsg in xs_host])  # batch-size groups + a remainder
    for v, ((xm, xsg), y) in enumerate(zip(xs_host, ys)):
        assert_same(hk.to_host(*y), oracle.matvec(kind, P, am, asg, xm, xsg),
                    f"kernel batch kind={kind} n={n} v={v}")
    # the stacked call directly, and a rejected vector inside a batch
    xm = torch.stack([hk.to_device(*xs_host[v])[0] for v in range(batch)])
    xsg = torch.stack([hk.to_device(*xs_host[v])[1] for v in range(batch)])
    if (n * gen.n_limbs(P)) % 2:  # vector 1 would start 8-byte aligned: the ABI rejects it
        with pytest.raises(hk.HKError):
            A.matvec_stacked(xm, xsg)
        return
    ym, ysg = A.matvec_stacked(xm, xsg)
    for v in range(batch):
        assert_same(hk.to_host(ym[v], ysg[v]), oracle.matvec(kind, P, am, asg, *xs_host[v]), f"stacked v={v}")
    bad = xsg.clone()
    bad[batch - 1, 0] = 2  # a sign outside {-1, 0, 1}
    with pytest.raises(hk.HKError):
        A.matvec_stacked(xm, bad)
