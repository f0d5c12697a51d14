"""paper_1402_5287_b200 -- exact multiprecision Hankel/Toeplitz/circulant matvec on B200.

Thin ctypes binding over the C ABI of ``include/hk.h`` (``lib/libhk.so``, built in-tree by
``_build.build()`` / ``__graft_entry__.build()``).  Every step of the product runs in the
library's CUDA kernels; this module only marshals torch tensors (device memory, the current
stream) into plain pointers.  There is NO CPU fallback: importing the package fails loudly when
the library is missing, and every call checks its status code.

Layout: a vector of ``count`` mantissas is ``mag`` uint64[count, L]
(limb 0 least significant, L = ceil(P/64)) + ``sign`` int8[count]; value = sign*mag*2^-P.
Outputs have Ly = 2L+1 limbs and value = sign*mag*2^-2P.  torch has limited uint64 support, so
magnitudes may be passed as torch.int64 or torch.uint64 (same bits).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB as _LIB_PATH

# dev A/B only (scripts/gpu_ab.sh): an alternative build of the same library, accepted only from
# this package's lib/ directory
_variant = os.environ.get("HK_LIB_VARIANT")
if _variant:
    _libdir = os.path.realpath(os.path.dirname(_LIB_PATH))
    if not os.path.realpath(_variant).startswith(_libdir + os.sep):
        raise ImportError(f"HK_LIB_VARIANT must name a build under {_libdir}")
    _LIB_PATH = _variant

HK_OK, HK_EINVAL, HK_ERANGE, HK_ENOMEM, HK_EUNSUPPORTED, HK_ECUDA = 0, -1, -2, -3, -4, -5
HANKEL, TOEPLITZ, CIRCULANT = 0, 1, 2
WS_STAGING = 1
WS_PREPARED = 2


class HKError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {status_string(code)} ({code})")


class PlanInfo(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("P", ctypes.c_int32), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("a_count", ctypes.c_int64), ("L", ctypes.c_int32),
                ("Ly", ctypes.c_int32), ("k_primes", ctypes.c_int32), ("w", ctypes.c_int32),
                ("Ls", ctypes.c_int32), ("log_n2", ctypes.c_int32), ("log_n1", ctypes.c_int32),
                ("cyclic", ctypes.c_int32), ("fold", ctypes.c_int32),
                ("margin_bits", ctypes.c_double), ("ws_bytes", ctypes.c_uint64),
                ("ws_bytes_staging", ctypes.c_uint64), ("ws_bytes_prepared", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class FftPlanInfo(ctypes.Structure):
    """hk_fft_plan_info (include/hk.h): the F3 FP64-FFT plan and its Percival bound."""
    _fields_ = [("kind", ctypes.c_int32), ("P", ctypes.c_int32), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("a_count", ctypes.c_int64), ("L", ctypes.c_int32),
                ("Ly", ctypes.c_int32), ("w", ctypes.c_int32), ("Ls", ctypes.c_int32),
                ("log_n1", ctypes.c_int32), ("log_n2", ctypes.c_int32), ("cyclic", ctypes.c_int32),
                ("fold", ctypes.c_int32), ("bound", ctypes.c_double), ("eps", ctypes.c_double),
                ("beta", ctypes.c_double), ("ws_bytes", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class ShardInfo(ctypes.Structure):
    """hk_shard_info (include/hk.h): sigma-coset sharding layout."""
    _fields_ = [("G", ctypes.c_int32), ("gamma", ctypes.c_int32), ("block_cols", ctypes.c_int64),
                ("rows_per_rank", ctypes.c_int64), ("y_rows", ctypes.c_int64),
                ("chunk_words", ctypes.c_int64), ("buffer_words", ctypes.c_int64),
                ("ws_bytes", ctypes.c_uint64), ("slice_chunk_words", ctypes.c_int64),
                ("slice_buffer_words", ctypes.c_int64), ("slice_rows_a", ctypes.c_int64),
                ("slice_rows_x", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"libhk.so not built ({_LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    sig = {
        "hk_limbs": (i32, [i32]),
        "hk_out_limbs": (i32, [i32]),
        "hk_status_string": (ctypes.c_char_p, [i32]),
        "hk_plan": (i32, [i32, i64, i64, i32, ctypes.POINTER(PlanInfo)]),
        "hk_workspace_size": (i32, [i32, i64, i64, i32, ctypes.c_uint32, ctypes.POINTER(sz)]),
        "hk_workspace_init": (i32, [i32, i64, i64, i32, ctypes.c_uint32, vp, sz, vp]),
        "hk_workspace_status": (i32, [vp, vp, ctypes.POINTER(i32)]),
        "hk_hankel_matvec": (i32, [i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_toeplitz_matvec": (i32, [i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_circulant_matvec": (i32, [i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_rect_matvec": (i32, [i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_matvec_host": (i32, [i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_matvec_host_async": (i32, [i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_schoolbook_matvec": (i32, [i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp]),
        "hk_matvec_stages": (i32, [i32, i64, i64, i32, ctypes.c_uint32, vp, vp, vp, vp, vp, vp,
                                   vp, sz, vp]),
        "hk_karatsuba_workspace_size": (i32, [i64, i32, i32, ctypes.POINTER(sz)]),
        "hk_prepare_a": (i32, [i32, i64, i64, i32, vp, vp, vp, sz, vp]),
        "hk_matvec_rounded": (i32, [i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_shard_plan": (i32, [i32, i64, i32, i32, ctypes.POINTER(ShardInfo)]),
        "hk_shard_workspace_init": (i32, [i32, i64, i32, i32, vp, sz, vp]),
        "hk_hankel_shard_forward": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_finish": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_forward_p2p": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_finish_p2p": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, vp, sz, vp]),
        "hk_matvec_prepared": (i32, [i32, i64, i64, i32, vp, vp, vp, vp, vp, sz, vp]),
        "hk_karatsuba_matvec": (i32, [i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_slice": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_slice_p2p": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_columns": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, sz, vp]),
        "hk_hankel_shard_columns_p2p": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, sz, vp]),
        "hk_batch_workspace_size": (i32, [i32, i64, i64, i32, i32, ctypes.POINTER(sz)]),
        "hk_batch_workspace_init": (i32, [i32, i64, i64, i32, i32, vp, sz, vp]),
        "hk_matvec_prepared_batch": (i32, [i32, i64, i64, i32, i32, vp, vp, vp, vp, vp, sz, vp]),
        "hk_fft_plan": (i32, [i32, i64, i32, ctypes.POINTER(FftPlanInfo)]),
        "hk_fft_workspace_init": (i32, [i32, i64, i32, vp, sz, vp]),
        "hk_fft_matvec": (i32, [i32, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "hk_fft_plan_w": (i32, [i32, i64, i32, i32, ctypes.POINTER(FftPlanInfo)]),
        "hk_fft_workspace_init_w": (i32, [i32, i64, i32, i32, vp, sz, vp]),
        "hk_fft_matvec_w": (i32, [i32, i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = ("hk_limbs", "hk_out_limbs", "hk_status_string", "hk_plan", "hk_workspace_size",
            "hk_workspace_init", "hk_workspace_status", "hk_hankel_matvec", "hk_toeplitz_matvec",
            "hk_circulant_matvec", "hk_hankel_rect_matvec", "hk_matvec_host", "hk_matvec_host_async",
            "hk_schoolbook_matvec", "hk_matvec_stages", "hk_karatsuba_workspace_size",
            "hk_karatsuba_matvec", "hk_prepare_a", "hk_matvec_prepared", "hk_shard_plan",
            "hk_shard_workspace_init", "hk_hankel_shard_forward", "hk_hankel_shard_finish",
            "hk_matvec_rounded", "hk_hankel_shard_forward_p2p", "hk_hankel_shard_finish_p2p",
            "hk_fft_plan", "hk_fft_workspace_init", "hk_fft_matvec", "hk_batch_workspace_size",
            "hk_batch_workspace_init", "hk_matvec_prepared_batch", "hk_hankel_shard_slice",
            "hk_hankel_shard_slice_p2p", "hk_hankel_shard_columns", "hk_hankel_shard_columns_p2p",
            "hk_fft_plan_w", "hk_fft_workspace_init_w", "hk_fft_matvec_w")
STAGE_SLICE_ROWS, STAGE_COLUMNS, STAGE_FINISH, STAGE_ALL = 1, 2, 4, 7


def library_path() -> str:
    return _LIB_PATH


def status_string(code: int) -> str:
    return _lib.hk_status_string(int(code)).decode()


def _check(code: int, where: str) -> None:
    if code != HK_OK:
        raise HKError(code, where)


def limbs(P: int) -> int:
    return int(_lib.hk_limbs(P))


def out_limbs(P: int) -> int:
    return int(_lib.hk_out_limbs(P))


def plan(kind: int, n: int, P: int, m: int | None = None) -> dict:
    """The exact plan (w, Ls, N1, N2, margin) the library uses; pure host call."""
    info = PlanInfo()
    _check(_lib.hk_plan(kind, n if m is None else m, n, P, ctypes.byref(info)), "hk_plan")
    return info.as_dict()


def workspace_size(kind: int, n: int, P: int, m: int | None = None, flags: int = 0) -> int:
    out = ctypes.c_size_t()
    _check(_lib.hk_workspace_size(kind, n if m is None else m, n, P, flags, ctypes.byref(out)),
           "hk_workspace_size")
    return int(out.value)


def _stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


class Workspace:
    """Caller-owned device workspace (a torch uint8 CUDA tensor) initialised for one problem."""

    def __init__(self, kind: int, n: int, P: int, m: int | None = None, flags: int = 0,
                 device=None, stream=None):
        import torch
        self.kind, self.n, self.P = int(kind), int(n), int(P)
        self.m = self.n if m is None else int(m)
        self.flags = int(flags)
        self.nbytes = workspace_size(kind, n, P, m=self.m, flags=flags)
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8,
                               device=device or torch.device("cuda", torch.cuda.current_device()))
        base = self.buf.data_ptr()
        self.ptr = (base + 255) & ~255
        _check(_lib.hk_workspace_init(kind, self.m, self.n, P, flags, self.ptr, self.nbytes,
                                      _stream_ptr(stream)), "hk_workspace_init")

    def status(self, stream=None) -> int:
        v = ctypes.c_int32()
        _check(_lib.hk_workspace_status(self.ptr, _stream_ptr(stream), ctypes.byref(v)),
               "hk_workspace_status")
        return int(v.value)

    def status_word(self):
        """The workspace header's data-status word (int32 at byte 16, include/hk.h) as a 1-element
        device tensor view, for stream-ordered copies of the status without a host sync."""
        import torch
        off = self.ptr - self.buf.data_ptr() + 16
        return self.buf[off:off + 4].view(torch.int32)


def _dev_ptr(t, dtypes, shape, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor")
    if t.dtype not in dtypes:
        raise TypeError(f"{name}: dtype {t.dtype} not in {dtypes}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return t.data_ptr()


def _mag_dtypes():
    import torch
    return (torch.int64, torch.uint64)


def _run(kind, a_mag, a_sign, x_mag, x_sign, P, m=None, out=None, ws=None, stream=None,
         check=True, rounded=False):
    import torch
    n = int(x_mag.shape[0])
    m = n if m is None else int(m)
    L = limbs(P)
    Ly = L + 1 if rounded else out_limbs(P)
    na = (n if kind == CIRCULANT else m + n - 1)
    args = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (n,), "x_sign")]
    if out is None:
        out = (torch.empty((m, Ly), dtype=a_mag.dtype, device=a_mag.device),
               torch.empty((m,), dtype=torch.int8, device=a_mag.device))
    args += [_dev_ptr(out[0], _mag_dtypes(), (m, Ly), "y_mag"),
             _dev_ptr(out[1], (torch.int8,), (m,), "y_sign")]
    if ws is None:
        ws = Workspace(kind, n, P, m=m, stream=stream)
    if (ws.kind, ws.m, ws.n, ws.P) != (kind, m, n, P):
        raise ValueError("workspace was initialised for a different problem")
    sp = _stream_ptr(stream)
    if rounded:
        rc = _lib.hk_matvec_rounded(kind, m, n, P, *args, ws.ptr, ws.nbytes, sp)
    elif kind == HANKEL and m != n:
        rc = _lib.hk_hankel_rect_matvec(m, n, P, *args, ws.ptr, ws.nbytes, sp)
    else:
        fn = {HANKEL: _lib.hk_hankel_matvec, TOEPLITZ: _lib.hk_toeplitz_matvec,
              CIRCULANT: _lib.hk_circulant_matvec}[kind]
        rc = fn(n, P, *args, ws.ptr, ws.nbytes, sp)
    _check(rc, "matvec")
    if check:
        _check(ws.status(stream), "matvec data status")
    return out


def hankel_matvec(a_mag, a_sign, x_mag, x_sign, P, out=None, ws=None, stream=None, check=True):
    """y = A_H x, A_H[i][j] = a_{i+j-1}; a has 2n-1 entries."""
    return _run(HANKEL, a_mag, a_sign, x_mag, x_sign, P, out=out, ws=ws, stream=stream, check=check)


def toeplitz_matvec(a_mag, a_sign, x_mag, x_sign, P, out=None, ws=None, stream=None, check=True):
    """y = A_T x, A_T[i][j] = a_{n-i+j}."""
    return _run(TOEPLITZ, a_mag, a_sign, x_mag, x_sign, P, out=out, ws=ws, stream=stream, check=check)


def circulant_matvec(c_mag, c_sign, x_mag, x_sign, P, out=None, ws=None, stream=None, check=True):
    """y = A_C x, A_C[i][j] = c_{((i-j) mod n)+1}."""
    return _run(CIRCULANT, c_mag, c_sign, x_mag, x_sign, P, out=out, ws=ws, stream=stream, check=check)


def hankel_rect_matvec(a_mag, a_sign, x_mag, x_sign, P, m, out=None, ws=None, stream=None,
                       check=True):
    """Rows 1..m of a Hankel product over the window a[0 .. m+n-2] (row-block shard)."""
    return _run(HANKEL, a_mag, a_sign, x_mag, x_sign, P, m=m, out=out, ws=ws, stream=stream,
                check=check)


def matvec(kind, a_mag, a_sign, x_mag, x_sign, P, m=None, out=None, ws=None, stream=None, check=True,
           rounded=False):
    """y = A x exactly (Ly = 2L+1 limbs, scale 2^-2P), or with ``rounded`` (F4, hk_matvec_rounded)
    rounded half-to-even back to the input format (L+1 limbs, scale 2^-P)."""
    return _run(kind, a_mag, a_sign, x_mag, x_sign, P, m=m, out=out, ws=ws, stream=stream, check=check,
                rounded=rounded)


def matvec_host(kind, a_mag, a_sign, x_mag, x_sign, P, m=None, out=None, ws=None, stream=None):
    """End-to-end call with HOST (numpy or pinned torch CPU) buffers through hk_matvec_host:
    H2D copies, the matvec and D2H copies happen inside the library call."""
    n = int(x_mag.shape[0])
    m = n if m is None else int(m)
    Ly = out_limbs(P)

    def hptr(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    if out is None:
        out = (np.empty((m, Ly), dtype=np.uint64), np.empty((m,), dtype=np.int8))
    if ws is None:
        ws = Workspace(kind, n, P, m=m, flags=WS_STAGING, stream=stream)
    if not ws.flags & WS_STAGING:
        raise ValueError("workspace needs WS_STAGING for host-buffer calls")
    rc = _lib.hk_matvec_host(kind, m, n, P, hptr(a_mag), hptr(a_sign), hptr(x_mag), hptr(x_sign),
                             hptr(out[0]), hptr(out[1]), ws.ptr, ws.nbytes, _stream_ptr(stream))
    _check(rc, "hk_matvec_host")
    return out


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return arr


def shard_forward_p2p(ws: ShardWorkspace, g, a_mag, a_sign, x_mag, x_sign, recv_ptrs, stream=None):
    """Phase 1 of rank g with the all-to-all fused into K2's stores: recv_ptrs[r] = rank r's receive
    buffer (device pointers mapped into this process, e.g. torch symmetric memory)."""
    import torch
    L, na = limbs(ws.P), (ws.n if ws.kind == CIRCULANT else 2 * ws.n - 1)
    if len(recv_ptrs) != ws.G:
        raise ValueError("need one receive-buffer pointer per rank")
    ptrs = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (ws.n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (ws.n,), "x_sign")]
    arr = _ptr_array(recv_ptrs)
    _check(_lib.hk_hankel_shard_forward_p2p(ws.kind, ws.n, ws.P, ws.G, int(g), *ptrs,
                                            ctypes.cast(arr, ctypes.c_void_p), ws.ptr, ws.nbytes,
                                            _stream_ptr(stream)), "hk_hankel_shard_forward_p2p")


def shard_finish_p2p(ws: ShardWorkspace, g, recv, y_mag_ptrs, y_sign_ptrs, stream=None):
    """Phase 2 of rank g with the y all-gather fused into K3's stores: y_*_ptrs[d] = rank d's padded
    y buffers (y_rows rows)."""
    import torch
    if len(y_mag_ptrs) != ws.G or len(y_sign_ptrs) != ws.G:
        raise ValueError("need one y pointer per rank")
    r = _dev_ptr(recv, (torch.int32,), (ws.info["buffer_words"],), "recv")
    am, asg = _ptr_array(y_mag_ptrs), _ptr_array(y_sign_ptrs)
    _check(_lib.hk_hankel_shard_finish_p2p(ws.kind, ws.n, ws.P, ws.G, int(g), r,
                                           ctypes.cast(am, ctypes.c_void_p),
                                           ctypes.cast(asg, ctypes.c_void_p), ws.ptr, ws.nbytes,
                                           _stream_ptr(stream)), "hk_hankel_shard_finish_p2p")


class HostPipeline:
    """Throughput over a stream of independent problems with HOST buffers (hk_matvec_host_async):
    ``depth`` lanes, each a CUDA stream with its own staging workspace; submit() enqueues a whole
    call (H2D of a and x, the matvec, D2H of y and of the data status) on the next lane, so one
    call's copies overlap other calls' kernels.  Host buffers should be pinned.  A lane is reused
    only after its previous call has completed (submit() waits for it)."""

    def __init__(self, kind, n, P, m=None, depth=3, device=None):
        import torch
        self.kind, self.n, self.P = int(kind), int(n), int(P)
        self.m = self.n if m is None else int(m)
        self.depth = int(depth)
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(self.depth)]
        self.ws = []
        for st in self.streams:
            self.ws.append(Workspace(kind, self.n, P, m=self.m, flags=WS_STAGING, stream=st))
        self.status = torch.zeros((self.depth,), dtype=torch.int32).pin_memory()
        self.events = [None] * self.depth
        self.k = 0
        torch.cuda.synchronize(dev)

    def submit(self, a_mag, a_sign, x_mag, x_sign, out):
        """Enqueue one call; out = (y_mag, y_sign) pinned host tensors.  Returns the lane index."""
        import torch
        lane = self.k % self.depth
        self.k += 1
        if self.events[lane] is not None:
            self.events[lane].synchronize()
            self._check_lane(lane)
        st, ws = self.streams[lane], self.ws[lane]

        def hptr(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

        rc = _lib.hk_matvec_host_async(self.kind, self.m, self.n, self.P, hptr(a_mag), hptr(a_sign),
                                       hptr(x_mag), hptr(x_sign), hptr(out[0]), hptr(out[1]),
                                       self.status.data_ptr() + 4 * lane, ws.ptr, ws.nbytes,
                                       st.cuda_stream)
        _check(rc, "hk_matvec_host_async")
        ev = torch.cuda.Event()
        ev.record(st)
        self.events[lane] = ev
        return lane

    def _check_lane(self, lane):
        code = int(self.status[lane].item())
        if code != HK_OK:
            raise HKError(code, "hk_matvec_host_async data status")

    def drain(self):
        """Wait for every call in flight and check their data status."""
        for lane, ev in enumerate(self.events):
            if ev is not None:
                ev.synchronize()
                self._check_lane(lane)
                self.events[lane] = None


# ---- sigma-coset sharding phases (include/hk.h; orchestration in paper_1402_5287_b200.dist)
def shard_plan(kind, n, P, G) -> dict:
    info = ShardInfo()
    _check(_lib.hk_shard_plan(int(kind), int(n), int(P), int(G), ctypes.byref(info)), "hk_shard_plan")
    return info.as_dict()


class ShardWorkspace:
    """Per-rank device workspace of the sigma-coset sharded path."""

    def __init__(self, kind, n, P, G, device=None, stream=None):
        import torch
        self.kind, self.n, self.P, self.G = int(kind), int(n), int(P), int(G)
        self.info = shard_plan(kind, n, P, G)
        self.nbytes = int(self.info["ws_bytes"])
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8,
                               device=device or torch.device("cuda", torch.cuda.current_device()))
        self.ptr = (self.buf.data_ptr() + 255) & ~255
        _check(_lib.hk_shard_workspace_init(self.kind, self.n, self.P, self.G, self.ptr, self.nbytes,
                                            _stream_ptr(stream)), "hk_shard_workspace_init")

    status_word = Workspace.status_word

    def status(self, stream=None) -> int:
        v = ctypes.c_int32()
        _check(_lib.hk_workspace_status(self.ptr, _stream_ptr(stream), ctypes.byref(v)),
               "hk_workspace_status")
        return int(v.value)


def shard_forward(ws: ShardWorkspace, g, a_mag, a_sign, x_mag, x_sign, send, stream=None):
    """Phase 1 of rank g: send (int32 CUDA tensor of buffer_words) <- G all-to-all chunks."""
    import torch
    L, na = limbs(ws.P), (ws.n if ws.kind == CIRCULANT else 2 * ws.n - 1)
    ptrs = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (ws.n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (ws.n,), "x_sign"),
            _dev_ptr(send, (torch.int32,), (ws.info["buffer_words"],), "send")]
    _check(_lib.hk_hankel_shard_forward(ws.kind, ws.n, ws.P, ws.G, int(g), *ptrs, ws.ptr,
                                        ws.nbytes, _stream_ptr(stream)), "hk_hankel_shard_forward")


def shard_slice(ws: ShardWorkspace, g, a_mag, a_sign, x_mag, x_sign, slice_send, stream=None):
    """Sliced phase 1a of rank g: K1 over this rank's matrix positions only, every sigma-block
    scattered into chunk d of slice_send (int32, slice_buffer_words, zero-initialised)."""
    import torch
    L, na = limbs(ws.P), (ws.n if ws.kind == CIRCULANT else 2 * ws.n - 1)
    ptrs = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (ws.n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (ws.n,), "x_sign"),
            _dev_ptr(slice_send, (torch.int32,), (ws.info["slice_buffer_words"],), "slice_send")]
    _check(_lib.hk_hankel_shard_slice(ws.kind, ws.n, ws.P, ws.G, int(g), *ptrs, ws.ptr, ws.nbytes,
                                      _stream_ptr(stream)), "hk_hankel_shard_slice")


def shard_slice_p2p(ws: ShardWorkspace, g, a_mag, a_sign, x_mag, x_sign, slice_recv_ptrs, stream=None):
    """Sliced phase 1a with the slice exchange fused into K1's stores: slice_recv_ptrs[d] = rank d's
    slice receive buffer (peer memory)."""
    import torch
    L, na = limbs(ws.P), (ws.n if ws.kind == CIRCULANT else 2 * ws.n - 1)
    if len(slice_recv_ptrs) != ws.G:
        raise ValueError("need one slice receive-buffer pointer per rank")
    ptrs = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (ws.n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (ws.n,), "x_sign")]
    arr = _ptr_array(slice_recv_ptrs)
    _check(_lib.hk_hankel_shard_slice_p2p(ws.kind, ws.n, ws.P, ws.G, int(g), *ptrs,
                                          ctypes.cast(arr, ctypes.c_void_p), ws.ptr, ws.nbytes,
                                          _stream_ptr(stream)), "hk_hankel_shard_slice_p2p")


def shard_columns(ws: ShardWorkspace, g, slice_recv, send, stream=None):
    """Sliced phase 1b of rank g: K2 on its columns gathered from slice_recv; output into send."""
    import torch
    r = _dev_ptr(slice_recv, (torch.int32,), (ws.info["slice_buffer_words"],), "slice_recv")
    sd = _dev_ptr(send, (torch.int32,), (ws.info["buffer_words"],), "send")
    _check(_lib.hk_hankel_shard_columns(ws.kind, ws.n, ws.P, ws.G, int(g), r, sd, ws.ptr, ws.nbytes,
                                        _stream_ptr(stream)), "hk_hankel_shard_columns")


def shard_columns_p2p(ws: ShardWorkspace, g, slice_recv, recv_ptrs, stream=None):
    """Sliced phase 1b with the all-to-all fused into K2's stores (recv_ptrs[d] = rank d's receive buffer)."""
    import torch
    if len(recv_ptrs) != ws.G:
        raise ValueError("need one receive-buffer pointer per rank")
    r = _dev_ptr(slice_recv, (torch.int32,), (ws.info["slice_buffer_words"],), "slice_recv")
    arr = _ptr_array(recv_ptrs)
    _check(_lib.hk_hankel_shard_columns_p2p(ws.kind, ws.n, ws.P, ws.G, int(g), r,
                                            ctypes.cast(arr, ctypes.c_void_p), ws.ptr, ws.nbytes,
                                            _stream_ptr(stream)), "hk_hankel_shard_columns_p2p")


def shard_finish(ws: ShardWorkspace, g, recv, y_mag, y_sign, stream=None):
    """Phase 2 of rank g: rows [g rpr, (g+1) rpr) of the padded y (y_rows rows) from recv."""
    import torch
    yr, Ly = ws.info["y_rows"], out_limbs(ws.P)
    ptrs = [_dev_ptr(recv, (torch.int32,), (ws.info["buffer_words"],), "recv"),
            _dev_ptr(y_mag, _mag_dtypes(), (yr, Ly), "y_mag"),
            _dev_ptr(y_sign, (torch.int8,), (yr,), "y_sign")]
    _check(_lib.hk_hankel_shard_finish(ws.kind, ws.n, ws.P, ws.G, int(g), *ptrs, ws.ptr, ws.nbytes,
                                       _stream_ptr(stream)), "hk_hankel_shard_finish")


class Problem:
    """A prepared device problem (inputs, output and workspace resident in HBM) for repeated
    calls; ``run(stages)`` launches the selected pipeline stages on the current stream."""

    def __init__(self, kind, a_mag, a_sign, x_mag, x_sign, P, m=None, stream=None):
        import torch
        self.kind, self.P = int(kind), int(P)
        self.n = int(x_mag.shape[0])
        self.m = self.n if m is None else int(m)
        L, Ly = limbs(P), out_limbs(P)
        na = (self.n if kind == CIRCULANT else self.m + self.n - 1)
        self.inputs = (a_mag, a_sign, x_mag, x_sign)
        self.ptrs = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
                     _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
                     _dev_ptr(x_mag, _mag_dtypes(), (self.n, L), "x_mag"),
                     _dev_ptr(x_sign, (torch.int8,), (self.n,), "x_sign")]
        self.y_mag = torch.empty((self.m, Ly), dtype=a_mag.dtype, device=a_mag.device)
        self.y_sign = torch.empty((self.m,), dtype=torch.int8, device=a_mag.device)
        self.ptrs += [self.y_mag.data_ptr(), self.y_sign.data_ptr()]
        self.ws = Workspace(kind, self.n, P, m=self.m, stream=stream)

    def run(self, stages: int = STAGE_ALL, stream=None) -> None:
        rc = _lib.hk_matvec_stages(self.kind, self.m, self.n, self.P, stages, *self.ptrs,
                                   self.ws.ptr, self.ws.nbytes, _stream_ptr(stream))
        _check(rc, "hk_matvec_stages")

    def capture(self):
        """Capture one whole step (all stages, this Problem's fixed buffers) in a CUDA graph on a
        side stream; replay() then relaunches it with one host call, which is what small problems
        are bound by (C1: ~30 us of host work per hk_matvec_stages call vs ~27 us on the GPU)."""
        import torch
        dev = self.y_mag.device
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            self.run(stream=s)  # first launch outside the capture (kernel attributes, plan cache)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.run(stream=s)
        torch.cuda.current_stream(dev).wait_stream(s)
        self._graph = g
        return self

    def replay(self) -> None:
        """Launch the captured step on the current stream (see capture())."""
        self._graph.replay()

    def status(self, stream=None) -> int:
        return self.ws.status(stream)

    def result(self):
        """(y_mag, y_sign) device tensors of the last run (overwritten by the next)."""
        return self.y_mag, self.y_sign


class BatchWorkspace:
    """A prepared workspace plus `nvec` per-vector transform regions (hk_batch_workspace_size/init)."""

    def __init__(self, kind, n, P, m=None, nvec=2, device=None, stream=None):
        import torch
        self.kind, self.n, self.P = int(kind), int(n), int(P)
        self.m = self.n if m is None else int(m)
        self.nvec = int(nvec)
        out = ctypes.c_size_t()
        _check(_lib.hk_batch_workspace_size(self.kind, self.m, self.n, self.P, self.nvec, ctypes.byref(out)),
               "hk_batch_workspace_size")
        self.nbytes = int(out.value)
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8,
                               device=device or torch.device("cuda", torch.cuda.current_device()))
        self.ptr = (self.buf.data_ptr() + 255) & ~255
        _check(_lib.hk_batch_workspace_init(self.kind, self.m, self.n, self.P, self.nvec, self.ptr,
                                            self.nbytes, _stream_ptr(stream)), "hk_batch_workspace_init")

    status = Workspace.status
    status_word = Workspace.status_word


class PreparedMatrix:
    """F1 (fixed-A repeated products, the paper's Lanczos use P:32-36): the 2-D transform of a is
    computed once (hk_prepare_a) and reused by every matvec(x) (hk_matvec_prepared)."""

    def __init__(self, kind, a_mag, a_sign, P, n, m=None, stream=None, check=True, lanes=1, batch=1):
        """lanes > 1: multi-vector batching for matvec_batch() -- that many CUDA streams, each with
        its own prepared workspace (a's transform computed once per lane), so several vectors'
        products are in flight at once and fill each other's partial last waves.
        batch > 1: kernel-level batching instead -- ONE prepared copy of a's transform and room for
        `batch` vectors; matvec_stacked() / matvec_batch() run up to `batch` vectors per launch of
        each kernel (hk_matvec_prepared_batch; every A^ column read from HBM once per batch)."""
        import torch
        self.kind, self.P, self.n = int(kind), int(P), int(n)
        self.m = self.n if m is None else int(m)
        self.batch = max(1, int(batch))
        if self.batch > 1 and int(lanes) > 1:
            raise ValueError("choose lanes (stream-level) or batch (kernel-level) batching, not both")
        L = limbs(P)
        na = (self.n if kind == CIRCULANT else self.m + self.n - 1)
        self.a = (a_mag, a_sign)
        pa = _dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag")
        ps = _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign")
        if self.batch > 1:
            self.ws = BatchWorkspace(kind, self.n, P, m=self.m, nvec=self.batch, stream=stream)
        else:
            self.ws = Workspace(kind, self.n, P, m=self.m, flags=WS_PREPARED, stream=stream)
        _check(_lib.hk_prepare_a(self.kind, self.m, self.n, self.P, pa, ps, self.ws.ptr,
                                 self.ws.nbytes, _stream_ptr(stream)), "hk_prepare_a")
        if check:
            _check(self.ws.status(stream), "hk_prepare_a data status")
        self.lanes = max(1, int(lanes))
        self._lane_ws, self._lane_st = [self.ws], [None]
        if self.lanes > 1:
            cur = torch.cuda.current_stream() if stream is None else stream
            for _ in range(self.lanes - 1):
                st = torch.cuda.Stream(device=a_mag.device)
                st.wait_stream(cur)
                ws = Workspace(kind, self.n, P, m=self.m, flags=WS_PREPARED, stream=st)
                _check(_lib.hk_prepare_a(self.kind, self.m, self.n, self.P, pa, ps, ws.ptr, ws.nbytes,
                                         st.cuda_stream), "hk_prepare_a")
                if check:
                    _check(ws.status(st), "hk_prepare_a data status")
                self._lane_ws.append(ws)
                self._lane_st.append(st)
            self._lane_st[0] = torch.cuda.Stream(device=a_mag.device)
            self._lane_st[0].wait_stream(cur)

    def matvec(self, x_mag, x_sign, out=None, stream=None, check=True):
        import torch
        L, Ly = limbs(self.P), out_limbs(self.P)
        px = _dev_ptr(x_mag, _mag_dtypes(), (self.n, L), "x_mag")
        pxs = _dev_ptr(x_sign, (torch.int8,), (self.n,), "x_sign")
        if out is None:
            out = (torch.empty((self.m, Ly), dtype=x_mag.dtype, device=x_mag.device),
                   torch.empty((self.m,), dtype=torch.int8, device=x_mag.device))
        py = _dev_ptr(out[0], _mag_dtypes(), (self.m, Ly), "y_mag")
        pys = _dev_ptr(out[1], (torch.int8,), (self.m,), "y_sign")
        _check(_lib.hk_matvec_prepared(self.kind, self.m, self.n, self.P, px, pxs, py, pys,
                                       self.ws.ptr, self.ws.nbytes, _stream_ptr(stream)),
               "hk_matvec_prepared")
        if check:
            _check(self.ws.status(stream), "hk_matvec_prepared data status")
        return out

    def matvec_stacked(self, x_mag, x_sign, out=None, stream=None, check=True):
        """Kernel-level batch: x_mag [v, n, L], x_sign [v, n] with v <= batch -> (y_mag [v, m, Ly],
        y_sign [v, m]) through hk_matvec_prepared_batch (one launch per kernel for all v)."""
        import torch
        if self.batch < 2:
            raise ValueError("matvec_stacked needs PreparedMatrix(..., batch=k), k > 1")
        L, Ly = limbs(self.P), out_limbs(self.P)
        v = int(x_mag.shape[0])
        if not 1 <= v <= self.batch:
            raise ValueError(f"at most {self.batch} vectors per call")
        px = _dev_ptr(x_mag, _mag_dtypes(), (v, self.n, L), "x_mag")
        pxs = _dev_ptr(x_sign, (torch.int8,), (v, self.n), "x_sign")
        if out is None:
            out = (torch.empty((v, self.m, Ly), dtype=x_mag.dtype, device=x_mag.device),
                   torch.empty((v, self.m), dtype=torch.int8, device=x_mag.device))
        py = _dev_ptr(out[0], _mag_dtypes(), (v, self.m, Ly), "y_mag")
        pys = _dev_ptr(out[1], (torch.int8,), (v, self.m), "y_sign")
        _check(_lib.hk_matvec_prepared_batch(self.kind, self.m, self.n, self.P, v, px, pxs, py, pys,
                                             self.ws.ptr, self.ws.nbytes, _stream_ptr(stream)),
               "hk_matvec_prepared_batch")
        if check:
            _check(self.ws.status(stream), "hk_matvec_prepared_batch data status")
        return out

    def matvec_batch(self, xs, outs=None, stream=None, check=True):
        """y_v = A x_v for a list of (x_mag, x_sign) pairs, distributed round-robin over the lanes
        (see __init__), or stacked into kernel-level batches of `batch` vectors; ordered after and
        before the calling stream.  Returns the list of outputs."""
        import torch
        L, Ly = limbs(self.P), out_limbs(self.P)
        cur = torch.cuda.current_stream() if stream is None else stream
        if self.batch > 1:
            res = []
            # stacked vectors must each start 16-byte aligned: n L even (else one vector per launch)
            step = self.batch if (self.n * L) % 2 == 0 else 1
            for g0 in range(0, len(xs), step):
                grp = xs[g0:g0 + step]
                ym, ys = self.matvec_stacked(torch.stack([xm for xm, _ in grp]),
                                             torch.stack([xsg for _, xsg in grp]), stream=cur, check=check)
                for v in range(len(grp)):
                    if outs is not None:
                        outs[g0 + v][0].copy_(ym[v])
                        outs[g0 + v][1].copy_(ys[v])
                        res.append(outs[g0 + v])
                    else:
                        res.append((ym[v], ys[v]))
            return res
        if self.lanes == 1:
            return [self.matvec(xm, xsg, out=None if outs is None else outs[v], stream=cur, check=check)
                    for v, (xm, xsg) in enumerate(xs)]
        for st in self._lane_st:
            st.wait_stream(cur)
        res = []
        # each call resets its lane's status word, so every call's status is copied into its own
        # device slot right after it, on its lane (checked once at the end)
        slots = torch.zeros((len(xs),), dtype=torch.int32, device=xs[0][0].device) if check else None
        for v, (xm, xsg) in enumerate(xs):
            lane = v % self.lanes
            st, ws = self._lane_st[lane], self._lane_ws[lane]
            px = _dev_ptr(xm, _mag_dtypes(), (self.n, L), "x_mag")
            pxs = _dev_ptr(xsg, (torch.int8,), (self.n,), "x_sign")
            if outs is None:  # allocated on the calling stream, used on the lane (record_stream below)
                out = (torch.empty((self.m, Ly), dtype=xm.dtype, device=xm.device),
                       torch.empty((self.m,), dtype=torch.int8, device=xm.device))
            else:
                out = outs[v]
            py = _dev_ptr(out[0], _mag_dtypes(), (self.m, Ly), "y_mag")
            pys = _dev_ptr(out[1], (torch.int8,), (self.m,), "y_sign")
            _check(_lib.hk_matvec_prepared(self.kind, self.m, self.n, self.P, px, pxs, py, pys,
                                           ws.ptr, ws.nbytes, st.cuda_stream), "hk_matvec_prepared")
            if check:
                with torch.cuda.stream(st):
                    slots[v:v + 1].copy_(ws.status_word())
            for t in (xm, xsg, out[0], out[1]):
                t.record_stream(st)
            res.append(out)
        for st in self._lane_st:
            cur.wait_stream(st)
        if check:
            codes = slots.cpu().tolist()  # ordered after every lane (cur waited for them)
            for v, code in enumerate(codes):
                if code != HK_OK:
                    raise HKError(int(code), f"hk_matvec_prepared data status (vector {v})")
        return res


def schoolbook_matvec(kind, a_mag, a_sign, x_mag, x_sign, P, m=None, out=None, stream=None):
    """Companion A6: direct schoolbook limb products on the GPU (no transform)."""
    import torch
    n = int(x_mag.shape[0])
    m = n if m is None else int(m)
    L, Ly = limbs(P), out_limbs(P)
    na = (n if kind == CIRCULANT else m + n - 1)
    args = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (n,), "x_sign")]
    if out is None:
        out = (torch.empty((m, Ly), dtype=a_mag.dtype, device=a_mag.device),
               torch.empty((m,), dtype=torch.int8, device=a_mag.device))
    args += [_dev_ptr(out[0], _mag_dtypes(), (m, Ly), "y_mag"),
             _dev_ptr(out[1], (torch.int8,), (m,), "y_sign")]
    _check(_lib.hk_schoolbook_matvec(kind, m, n, P, *args, _stream_ptr(stream)),
           "hk_schoolbook_matvec")
    return out


def karatsuba_workspace_size(n: int, P: int, cutoff: int = 8) -> int:
    out = ctypes.c_size_t()
    _check(_lib.hk_karatsuba_workspace_size(n, P, cutoff, ctypes.byref(out)),
           "hk_karatsuba_workspace_size")
    return int(out.value)


def karatsuba_matvec(a_mag, a_sign, x_mag, x_sign, P, cutoff: int = 8, out=None, stream=None):
    """Companion A5: Algorithm 1 level by level on the GPU (Hankel)."""
    import torch
    n = int(x_mag.shape[0])
    L, Ly = limbs(P), out_limbs(P)
    args = [_dev_ptr(a_mag, _mag_dtypes(), (2 * n - 1, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (2 * n - 1,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (n,), "x_sign")]
    if out is None:
        out = (torch.empty((n, Ly), dtype=a_mag.dtype, device=a_mag.device),
               torch.empty((n,), dtype=torch.int8, device=a_mag.device))
    args += [_dev_ptr(out[0], _mag_dtypes(), (n, Ly), "y_mag"),
             _dev_ptr(out[1], (torch.int8,), (n,), "y_sign")]
    nbytes = karatsuba_workspace_size(n, P, cutoff)
    buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=a_mag.device)
    ptr = (buf.data_ptr() + 255) & ~255
    _check(_lib.hk_karatsuba_matvec(n, P, cutoff, *args, ptr, nbytes, _stream_ptr(stream)),
           "hk_karatsuba_matvec")
    # buf goes back to torch's caching allocator when this function returns; it was allocated on
    # the current stream, so tell the allocator the work on `stream` still uses it
    if stream is not None:
        buf.record_stream(stream)
    return out


# ---- F3: the paper's decomposition approach with a double-precision FFT (exact by Percival's bound)
def fft_plan(kind: int, n: int, P: int, w: int = 0) -> dict:
    """The FP64-FFT plan (digit width w, lengths, Percival bound); pure host call.  w > 0 forces
    the digit width (F3 accuracy study, hk_fft_plan_w: the bound may then exceed 1/2)."""
    info = FftPlanInfo()
    _check(_lib.hk_fft_plan_w(int(kind), int(n), int(P), int(w), ctypes.byref(info)), "hk_fft_plan_w")
    return info.as_dict()


class FftWorkspace:
    """Device workspace of the F3 path (twiddle tables, carry table, 2 x N1 x N2 complex doubles);
    w > 0: the forced-width plan of the accuracy study."""

    def __init__(self, kind, n, P, device=None, stream=None, w=0):
        import torch
        self.kind, self.n, self.P, self.w = int(kind), int(n), int(P), int(w)
        self.info = fft_plan(kind, n, P, w)
        self.nbytes = int(self.info["ws_bytes"])
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8,
                               device=device or torch.device("cuda", torch.cuda.current_device()))
        self.ptr = (self.buf.data_ptr() + 255) & ~255
        _check(_lib.hk_fft_workspace_init_w(self.kind, self.n, self.P, self.w, self.ptr, self.nbytes,
                                            _stream_ptr(stream)), "hk_fft_workspace_init_w")

    status = Workspace.status


def fft_matvec(kind, a_mag, a_sign, x_mag, x_sign, P, out=None, ws=None, stream=None, check=True,
               w=0, residual=None):
    """y = A x exactly through the FP64 FFT path (hk_fft_matvec): same layouts as matvec().

    Accuracy study (hk_fft_matvec_w): ``w`` > 0 forces the digit width -- past the proven one the
    result is not guaranteed exact; ``residual``, a zeroed float64 CUDA tensor of one element, is
    raised to the largest |v - rint(v)| over the rounded output coefficients."""
    import torch
    n = int(x_mag.shape[0])
    L, Ly = limbs(P), out_limbs(P)
    na = n if kind == CIRCULANT else 2 * n - 1
    args = [_dev_ptr(a_mag, _mag_dtypes(), (na, L), "a_mag"),
            _dev_ptr(a_sign, (torch.int8,), (na,), "a_sign"),
            _dev_ptr(x_mag, _mag_dtypes(), (n, L), "x_mag"),
            _dev_ptr(x_sign, (torch.int8,), (n,), "x_sign")]
    if out is None:
        out = (torch.empty((n, Ly), dtype=a_mag.dtype, device=a_mag.device),
               torch.empty((n,), dtype=torch.int8, device=a_mag.device))
    args += [_dev_ptr(out[0], _mag_dtypes(), (n, Ly), "y_mag"),
             _dev_ptr(out[1], (torch.int8,), (n,), "y_sign")]
    if ws is None:
        ws = FftWorkspace(kind, n, P, stream=stream, w=w)
    if (ws.kind, ws.n, ws.P, ws.w) != (int(kind), n, int(P), int(w)):
        raise ValueError("FFT workspace was initialised for a different problem")
    rp = None
    if residual is not None:
        rp = _dev_ptr(residual, (torch.float64,), (1,), "residual")
    _check(_lib.hk_fft_matvec_w(int(kind), n, int(P), int(w), *args, ws.ptr, ws.nbytes, _stream_ptr(stream),
                                rp), "hk_fft_matvec_w")
    if check:
        _check(ws.status(stream), "hk_fft_matvec data status")
    return out


def to_device(mag: np.ndarray, sign: np.ndarray, device="cuda"):
    """numpy (uint64 limbs, int8 signs) -> torch CUDA tensors (int64 view of the limbs)."""
    import torch
    m = torch.from_numpy(np.ascontiguousarray(mag).view(np.int64)).to(device)
    s = torch.from_numpy(np.ascontiguousarray(sign, dtype=np.int8)).to(device)
    return m, s


def to_host(mag, sign) -> tuple[np.ndarray, np.ndarray]:
    return (mag.cpu().numpy().view(np.uint64), sign.cpu().numpy())
