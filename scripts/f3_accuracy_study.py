"""F3 accuracy study with the library's own FP64 FFT kernels (second half).

PAPER.md P:169 leaves open "whether the loss of accuracy occurs in practice" for the decomposition
approach with a standard FFT.  hk_fft_matvec_w runs the F3 path at a FORCED balanced digit width w;
for every BASELINE config this sweeps w from the width Percival's bound proves exact upwards and
records, per w: the bound, the measured max |v - rint(v)| over every rounded output coefficient,
and whether y is still bit-identical to the NTT path's y (itself bit-identical to the oracle: the
committed digests of tests/test_gpu_digests.py), plus the time per matvec.  Inputs: the config's
own recipe (uniform, or carry-stress for C5) and, built for each w, equal positive entries whose
balanced digits all have (almost) the largest magnitude 2^(w-1) -- no cancellation, the norms the
bound assumes.  (All-ones mantissas are NOT a worst case here: in balanced digits 2^P - 1 is almost
all zeros.)
Usage: python scripts/f3_accuracy_study.py [configs...] > profiles/r02/f3_accuracy_study.log"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402


def max_digits(kind, n, P, w):
    """Every entry = sum_{t < floor(P/w)} 2^(w-1) 2^(w t) (< 2^P), sign +1: each w-bit chunk is
    2^(w-1), so every balanced digit is -2^(w-1) + 1 (the largest magnitude but one) and no
    coefficient sum cancels -- the case the bound's norms describe, built anew for each w."""
    L = (P + 63) // 64
    T = P // w
    m = sum(1 << (w - 1 + w * t) for t in range(T))
    row = np.array([(m >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(L)], dtype=np.uint64)
    na = n if kind == gen.CIRCULANT else 2 * n - 1
    am = np.ascontiguousarray(np.broadcast_to(row, (na, L)))
    xm = np.ascontiguousarray(np.broadcast_to(row, (n, L)))
    return am, np.ones(na, dtype=np.int8), xm, np.ones(n, dtype=np.int8)


def run_w(kind, n, P, w, inputs):
    """(plan, max residual, rows differing from the NTT path's y, ms per matvec) at digit width w."""
    am, asg, xm, xsg = inputs
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    ref_m, ref_s = hk.matvec(kind, a, sa, x, sx, P)  # NTT path: bit-exact vs the oracle
    info = hk.fft_plan(kind, n, P, w=w)
    ws = hk.FftWorkspace(kind, n, P, w=w)
    res = torch.zeros(1, dtype=torch.float64, device=a.device)
    ym, ys = hk.fft_matvec(kind, a, sa, x, sx, P, ws=ws, w=w, residual=res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        hk.fft_matvec(kind, a, sa, x, sx, P, out=(ym, ys), ws=ws, w=w, check=False)
    e1.record()
    torch.cuda.synchronize()
    bad = int(((ym != ref_m).any(dim=1) | (ys != ref_s)).nonzero().numel())
    return info, float(res.item()), bad, e0.elapsed_time(e1) / 3


def study(name, recipe_name, kind, n, P, make, max_extra=14):
    proven = hk.fft_plan(kind, n, P)
    fails = 0
    for w in range(proven["w"], proven["w"] + max_extra + 1):
        try:
            hk.fft_plan(kind, n, P, w=w)
        except hk.HKError:
            break
        info, r, bad, ms = run_w(kind, n, P, w, make(w))
        rec = {"config": name, "inputs": recipe_name, "n": n, "P": P, "w": w, "proven_w": proven["w"],
               "Ls": info["Ls"], "N1": 1 << info["log_n1"], "N2": 1 << info["log_n2"],
               "percival_bound": info["bound"], "max_residual": r, "exact": bad == 0,
               "rows_differing": bad, "ms_per_matvec": ms}
        print(json.dumps(rec), flush=True)
        fails = fails + 1 if bad else 0
        if fails >= 2:
            break


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C5T", "C5C"]
    for name in names:
        c = gen.CONFIGS[name]
        kind, n, P = c["kind"], c["n"], c["P"]
        inputs = gen.make_inputs(kind, n, P, c["seed"], c["recipe"])
        study(name, c["recipe"], kind, n, P, lambda w: inputs)
        study(name, "max_digits", kind, n, P, lambda w: max_digits(kind, n, P, w))


if __name__ == "__main__":
    main()
