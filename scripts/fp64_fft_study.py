"""F3 study: the paper's decomposition approach with a double-precision FFT
(PAPER.md P:119-170), measured on B200 -- "whether the loss of accuracy occurs in practice".

Not a product path.  For a BASELINE-shaped problem and slice width w, the mantissas are cut into
w-bit signed digits, the exact 2-D convolution over (matrix index x slice) of DESIGN.md section 3 is
computed with a complex FP64 FFT (torch.fft / cuFFT on the GPU), and we record
  * max |c - round(c)| over all needed output coefficients (the rounding residual; >= 0.5 means a
    wrong integer somewhere),
  * whether the carried, rounded result equals the exact y of the CUDA NTT path (libhk, itself
    bit-exact vs the oracle in tests/) on sampled rows,
  * the FP64 FFT convolution time on the device.
A rigorous a-priori bound (Percival 2003: N ||a||_2 ||x||_2 (3 log2 N + 1) ~ 3.3 eps < 1/2) cannot hold
at these sizes for any w: it needs Ls 2^w < 2^9.2 at C3 (F3).  This study measures the
error actually incurred.

usage: python scripts/fp64_fft_study.py [--configs C1,C2,C3] [--ws 8,10,12,14,16]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402


def digits(mag: np.ndarray, sign: np.ndarray, P: int, w: int) -> np.ndarray:
    """[rows, Ls] float64 signed digits sign * floor(|m| / 2^(w t)) mod 2^w."""
    rows, L = mag.shape
    Ls = -(-P // w)
    bits = np.unpackbits(mag.view(np.uint8).reshape(rows, L * 8), axis=1, bitorder="little")
    bits = bits[:, :P].astype(np.int64)
    pad = Ls * w - P
    if pad:
        bits = np.concatenate([bits, np.zeros((rows, pad), dtype=np.int64)], axis=1)
    d = (bits.reshape(rows, Ls, w) << np.arange(w, dtype=np.int64)).sum(axis=2)
    return (d * sign.astype(np.int64)[:, None]).astype(np.float64)


def limbs_to_int(row) -> int:
    v = 0
    for k, x in enumerate(row):
        v |= int(x) << (64 * k)
    return v


def run(cfg: str, w: int, sample_rows: int = 16) -> dict:
    c = gen.CONFIGS[cfg]
    kind, n, P = c["kind"], c["n"], c["P"]
    assert kind == gen.HANKEL
    am, asg, xm, xsg = gen.config_inputs(cfg)
    Ls = -(-P // w)
    N1 = 1 << math.ceil(math.log2(2 * n - 1))
    N2 = 1 << math.ceil(math.log2(2 * Ls - 1))
    dev = torch.device("cuda")
    A = torch.zeros((N1, N2), dtype=torch.complex128, device=dev)
    X = torch.zeros((N1, N2), dtype=torch.complex128, device=dev)
    A[: 2 * n - 1, :Ls] = torch.from_numpy(digits(am, asg, P, w)).to(dev)
    X[:n, :Ls] = torch.from_numpy(digits(xm, xsg, P, w)[::-1].copy()).to(dev)  # x reversed
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    C = torch.fft.ifft2(torch.fft.fft2(A) * torch.fft.fft2(X)).real[n - 1: 2 * n - 1, : 2 * Ls - 1]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    R = torch.round(C)
    resid = float((C - R).abs().max())
    # exact y from the CUDA NTT path (bit-exact vs the oracle in tests/)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ym, ys = hk.to_host(*hk.matvec(kind, a, sa, x, sx, P))
    rows = np.unique(np.linspace(0, n - 1, min(n, sample_rows)).astype(np.int64))
    Rh = R[torch.from_numpy(rows).to(dev)].cpu().numpy()
    exact = True
    for k, i in enumerate(rows):
        Y = sum(int(v) << (w * s) for s, v in enumerate(Rh[k]))
        want = limbs_to_int(ym[i]) * int(ys[i])
        exact &= (Y == want)
    del A, X, C, R
    torch.cuda.empty_cache()
    return {"config": cfg, "n": n, "P": P, "w": w, "Ls": Ls, "N1": N1, "N2": N2,
            "max_rounding_residual": resid, "bits_of_margin": (-math.log2(resid / 0.5) if resid > 0 else None),
            "rows_checked": int(len(rows)), "rounded_result_exact": bool(exact),
            "max_coeff_bits": 2 * w + math.log2(n * Ls), "fft_conv_ms": ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3")
    ap.add_argument("--ws", default="8,10,12,14,16")
    args = ap.parse_args()
    for cfg in args.configs.split(","):
        for w in map(int, args.ws.split(",")):
            t0 = time.time()
            r = run(cfg, w)
            r["wall_s"] = round(time.time() - t0, 1)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
