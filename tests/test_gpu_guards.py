"""Guard-band memory checks of every device entry point (stand-in for compute-sanitizer memcheck,
which this GPU pool refuses to run: profiles/r02/sanitizer_unavailable.txt).

Every device buffer a call touches -- the inputs a, x and their signs, the outputs y and their
signs, the caller-owned workspace -- is carved out of a larger allocation with GUARD bytes of a
canary pattern on each side.  After the call (and a synchronise) the test requires
  * every canary byte intact (no out-of-bounds write below or above any buffer),
  * the inputs byte-identical to what was uploaded (the C ABI declares them const),
  * y equal to the oracle's, element by element (PAPER.md P:50-90 defines the product),
at ragged sizes that leave partial tiles in every kernel (K1 row tiles, K2 columns, K3 row tiles,
the schoolbook's row clusters, the Karatsuba levels, the FP64-FFT path).  Reads out of bounds are
not detected this way; writes are, on every byte the guards cover.
"""
import ctypes

import numpy as np
import pytest

import hkinputs as gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GUARD = 1 << 16  # bytes of canary on each side of every buffer
CANARY = 0xA5


@pytest.fixture(scope="module")
def hk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1402_5287_b200 as hk
    return hk


class Guarded:
    """A device buffer of `nbytes` at a 256-byte aligned offset inside a canary-filled allocation."""

    def __init__(self, nbytes: int, init: np.ndarray | None = None):
        self.nbytes = int(nbytes)
        self.raw = torch.full((GUARD + self.nbytes + GUARD + 256,), CANARY, dtype=torch.uint8,
                              device="cuda")
        base = self.raw.data_ptr()
        self.off = GUARD + ((-(base + GUARD)) % 256)
        self.ptr = base + self.off
        self.view = self.raw[self.off:self.off + self.nbytes]
        if init is not None:
            b = np.ascontiguousarray(init).view(np.uint8).reshape(-1)
            assert b.size == self.nbytes
            self.view.copy_(torch.from_numpy(b.copy()))
            self.init = b.copy()
        else:
            self.init = None

    def check(self, what: str) -> None:
        h = self.raw.cpu().numpy()
        lo, hi = h[:self.off], h[self.off + self.nbytes:]
        bad_lo = np.nonzero(lo != CANARY)[0]
        bad_hi = np.nonzero(hi != CANARY)[0]
        assert bad_lo.size == 0, f"{what}: {bad_lo.size} bytes written below the buffer (last at -{self.off - bad_lo[-1]})"
        assert bad_hi.size == 0, f"{what}: {bad_hi.size} bytes written past the end (first at +{bad_hi[0]})"
        if self.init is not None:
            body = h[self.off:self.off + self.nbytes]
            assert np.array_equal(body, self.init), f"{what}: a const input was modified"

    def host(self, dtype, shape):
        return self.view.cpu().numpy().view(dtype).reshape(shape)


def _inputs(kind, n, P, seed, m=None):
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed, m=m)
    bufs = dict(am=Guarded(am.nbytes, am), asg=Guarded(asg.nbytes, asg),
                xm=Guarded(xm.nbytes, xm), xsg=Guarded(xsg.nbytes, xsg))
    return (am, asg, xm, xsg), bufs


def _outputs(rows, limbs):
    return dict(ym=Guarded(rows * limbs * 8), ysg=Guarded(rows))


def _check_all(bufs, what):
    torch.cuda.synchronize()
    for k, b in bufs.items():
        b.check(f"{what} [{k}]")


def _status(hk, ws_ptr, s):
    v = ctypes.c_int32()
    assert hk._lib.hk_workspace_status(ws_ptr, s, ctypes.byref(v)) == hk.HK_OK
    return v.value


SIZES = [(0, 37, 1000), (1, 300, 5000), (2, 129, 3328), (0, 1041, 700), (0, 90, 33216)]


@pytest.mark.parametrize("kind,n,P", SIZES)
def test_guarded_matvec(hk, kind, n, P):
    """hk_hankel / toeplitz / circulant_matvec: K1, K2, K3 write only their own buffers."""
    s = torch.cuda.current_stream().cuda_stream
    (am, asg, xm, xsg), bufs = _inputs(kind, n, P, seed=700 + n)
    Ly = gen.n_out_limbs(P)
    bufs.update(_outputs(n, Ly))
    wsb = hk.workspace_size(kind, n, P)
    bufs["ws"] = ws = Guarded(wsb)
    assert hk._lib.hk_workspace_init(kind, n, n, P, 0, ws.ptr, wsb, s) == hk.HK_OK
    fn = (hk._lib.hk_hankel_matvec, hk._lib.hk_toeplitz_matvec, hk._lib.hk_circulant_matvec)[kind]
    b = bufs
    for rep in range(2):  # a second call on the same workspace (reuse)
        rc = fn(n, P, b["am"].ptr, b["asg"].ptr, b["xm"].ptr, b["xsg"].ptr, b["ym"].ptr,
                b["ysg"].ptr, ws.ptr, wsb, s)
        assert rc == hk.HK_OK
        _check_all(bufs, f"matvec kind={kind} n={n} P={P} call {rep}")
    assert _status(hk, ws.ptr, s) == hk.HK_OK
    wm, wsg = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert np.array_equal(b["ym"].host(np.uint64, (n, Ly)), wm)
    assert np.array_equal(b["ysg"].host(np.int8, (n,)), wsg)


@pytest.mark.parametrize("m,n,P", [(13, 40, 1000), (200, 333, 4000)])
def test_guarded_rect_and_rounded(hk, m, n, P):
    """hk_hankel_rect_matvec (row window) and hk_matvec_rounded (F4) in guarded buffers."""
    s = torch.cuda.current_stream().cuda_stream
    (am, asg, xm, xsg), bufs = _inputs(0, n, P, seed=900 + m, m=m)
    Ly, L = gen.n_out_limbs(P), gen.n_limbs(P)
    bufs.update(_outputs(m, Ly))
    wsb = hk.workspace_size(0, n, P, m=m)
    bufs["ws"] = ws = Guarded(wsb)
    assert hk._lib.hk_workspace_init(0, m, n, P, 0, ws.ptr, wsb, s) == hk.HK_OK
    b = bufs
    assert hk._lib.hk_hankel_rect_matvec(m, n, P, b["am"].ptr, b["asg"].ptr, b["xm"].ptr, b["xsg"].ptr,
                                         b["ym"].ptr, b["ysg"].ptr, ws.ptr, wsb, s) == hk.HK_OK
    _check_all(bufs, f"rect m={m} n={n}")
    wm, wsg = oracle.matvec(0, P, am, asg, xm, xsg, m=m)
    assert np.array_equal(b["ym"].host(np.uint64, (m, Ly)), wm)
    assert np.array_equal(b["ysg"].host(np.int8, (m,)), wsg)
    r = _outputs(m, L + 1)
    assert hk._lib.hk_matvec_rounded(0, m, n, P, b["am"].ptr, b["asg"].ptr, b["xm"].ptr, b["xsg"].ptr,
                                     r["ym"].ptr, r["ysg"].ptr, ws.ptr, wsb, s) == hk.HK_OK
    _check_all({**bufs, **{"r" + k: v for k, v in r.items()}}, f"rounded m={m} n={n}")
    assert _status(hk, ws.ptr, s) == hk.HK_OK


@pytest.mark.parametrize("kind,n,P", [(0, 77, 2000), (2, 64, 1500)])
def test_guarded_prepared_and_host(hk, kind, n, P):
    """hk_prepare_a + hk_matvec_prepared (F1) and hk_matvec_host (staging area) in guarded buffers."""
    s = torch.cuda.current_stream().cuda_stream
    (am, asg, xm, xsg), bufs = _inputs(kind, n, P, seed=1300 + n)
    Ly = gen.n_out_limbs(P)
    bufs.update(_outputs(n, Ly))
    # the two flags are exclusive (the prepared transform and the staging area share the space
    # after the base layout, include/hk.h): one workspace per entry point
    wsb = hk.workspace_size(kind, n, P, flags=hk.WS_PREPARED)
    bufs["ws"] = ws = Guarded(wsb)
    assert hk._lib.hk_workspace_init(kind, n, n, P, hk.WS_PREPARED, ws.ptr, wsb, s) == hk.HK_OK
    b = bufs
    assert hk._lib.hk_prepare_a(kind, n, n, P, b["am"].ptr, b["asg"].ptr, ws.ptr, wsb, s) == hk.HK_OK
    assert hk._lib.hk_matvec_prepared(kind, n, n, P, b["xm"].ptr, b["xsg"].ptr, b["ym"].ptr, b["ysg"].ptr,
                                      ws.ptr, wsb, s) == hk.HK_OK
    _check_all(bufs, f"prepared kind={kind} n={n}")
    wm, wsg = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert np.array_equal(b["ym"].host(np.uint64, (n, Ly)), wm)
    assert np.array_equal(b["ysg"].host(np.int8, (n,)), wsg)
    # host buffers: the device side touched is the workspace (staging) only
    hsb = hk.workspace_size(kind, n, P, flags=hk.WS_STAGING)
    hws = Guarded(hsb)
    assert hk._lib.hk_workspace_init(kind, n, n, P, hk.WS_STAGING, hws.ptr, hsb, s) == hk.HK_OK
    yh = np.zeros((n, Ly), dtype=np.uint64)
    ysh = np.zeros(n, dtype=np.int8)
    rc = hk._lib.hk_matvec_host(kind, n, n, P, am.ctypes.data, asg.ctypes.data, xm.ctypes.data,
                                xsg.ctypes.data, yh.ctypes.data, ysh.ctypes.data, hws.ptr, hsb, s)
    assert rc == hk.HK_OK
    hws.check("host call [ws]")
    _check_all(bufs, f"host call kind={kind} n={n}")
    assert np.array_equal(yh, wm) and np.array_equal(ysh, wsg)


@pytest.mark.parametrize("kind,n,P", [(0, 45, 1200), (1, 200, 4100)])
def test_guarded_schoolbook_and_fft(hk, kind, n, P):
    """A6 schoolbook (no workspace) and the F3 FP64-FFT path in guarded buffers."""
    s = torch.cuda.current_stream().cuda_stream
    (am, asg, xm, xsg), bufs = _inputs(kind, n, P, seed=1700 + n)
    Ly = gen.n_out_limbs(P)
    bufs.update(_outputs(n, Ly))
    b = bufs
    wm, wsg = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert hk._lib.hk_schoolbook_matvec(kind, n, n, P, b["am"].ptr, b["asg"].ptr, b["xm"].ptr,
                                        b["xsg"].ptr, b["ym"].ptr, b["ysg"].ptr, s) == hk.HK_OK
    _check_all(bufs, f"schoolbook kind={kind} n={n}")
    assert np.array_equal(b["ym"].host(np.uint64, (n, Ly)), wm)
    info = hk.FftPlanInfo()
    assert hk._lib.hk_fft_plan(kind, n, P, ctypes.byref(info)) == hk.HK_OK
    f = _outputs(n, Ly)
    f["ws"] = fws = Guarded(int(info.ws_bytes))
    assert hk._lib.hk_fft_workspace_init(kind, n, P, fws.ptr, fws.nbytes, s) == hk.HK_OK
    assert hk._lib.hk_fft_matvec(kind, n, P, b["am"].ptr, b["asg"].ptr, b["xm"].ptr, b["xsg"].ptr,
                                 f["ym"].ptr, f["ysg"].ptr, fws.ptr, fws.nbytes, s) == hk.HK_OK
    _check_all({**bufs, **{"fft_" + k: v for k, v in f.items()}}, f"fft kind={kind} n={n}")
    assert _status(hk, fws.ptr, s) == hk.HK_OK
    assert np.array_equal(f["ym"].host(np.uint64, (n, Ly)), wm)
    assert np.array_equal(f["ysg"].host(np.int8, (n,)), wsg)


@pytest.mark.parametrize("n,P,cutoff", [(37, 700, 4), (100, 2000, 8)])
def test_guarded_karatsuba(hk, n, P, cutoff):
    """A5 Karatsuba-like levels: every level's operands stay inside the sized workspace."""
    s = torch.cuda.current_stream().cuda_stream
    (am, asg, xm, xsg), bufs = _inputs(0, n, P, seed=2100 + n)
    Ly = gen.n_out_limbs(P)
    bufs.update(_outputs(n, Ly))
    sz = ctypes.c_size_t()
    assert hk._lib.hk_karatsuba_workspace_size(n, P, cutoff, ctypes.byref(sz)) == hk.HK_OK
    bufs["ws"] = ws = Guarded(int(sz.value))
    b = bufs
    assert hk._lib.hk_karatsuba_matvec(n, P, cutoff, b["am"].ptr, b["asg"].ptr, b["xm"].ptr, b["xsg"].ptr,
                                       b["ym"].ptr, b["ysg"].ptr, ws.ptr, ws.nbytes, s) == hk.HK_OK
    _check_all(bufs, f"karatsuba n={n} cutoff={cutoff}")
    wm, wsg = oracle.matvec(0, P, am, asg, xm, xsg)
    assert np.array_equal(b["ym"].host(np.uint64, (n, Ly)), wm)
    assert np.array_equal(b["ysg"].host(np.int8, (n,)), wsg)
