#!/usr/bin/env python
"""Evidence for the companion kernels (north_star: "each choice evidenced by
ncu counters"): CUDA-event times of hk_schoolbook_matvec (A6), hk_karatsuba_matvec (A5) and the
NTT path on the same seeded Hankel inputs, with each method's algorithmic work rate:
  A6: 32x32->64-bit limb products  n^2 L32^2 (exact count: every (i, j) pair, full L32 x L32)
  A5: the same limb products at its leaves, from the recurrence M(n) = 2 M(m) + M(m1), M(<=c) = c^2
      (Algorithm 1), leaf entries W = L + 1 limbs
Results agree bit for bit between methods (checked).  The A6 inner loop issues one IMAD.WIDE (quarter
rate: 32 lanes/clk/SM, profiles/r01/micro_pipes.log) per limb product, so its pipe peak is
148 x 32 x f_sm products/s.  ncu --set full captures of k6_schoolbook / k5_leaf are taken by
scripts/gpu_companions.sh.

usage: python scripts/companions_profile.py [--cases 64:3328,256:3328,128:33216]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402


def timeit(fn, reps):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def karatsuba_leaf_products(n, cutoff):
    """Number of size-c leaf matvecs' entry products: M(n) = 2 M(m) + M(m1), M(s) = s^2 for s <= cutoff
    (Algorithm 1, m = floor(n/2), m1 = n - m)."""
    memo = {}

    def M(s):
        if s <= cutoff:
            return s * s
        if s in memo:
            return memo[s]
        m = s // 2
        v = 2 * M(m) + M(s - m)
        memo[s] = v
        return v
    return M(n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="64:3328,256:3328,128:33216")
    ap.add_argument("--cutoff", type=int, default=8)
    args = ap.parse_args()
    props = torch.cuda.get_device_properties(0)
    f_sm = float(os.environ.get("HK_SM_MHZ", "1965")) * 1e6
    wide_peak = props.multi_processor_count * 32 * f_sm  # IMAD.WIDE lanes/s
    for case in args.cases.split(","):
        n, P = map(int, case.split(":"))
        am, asg, xm, xsg = gen.make_inputs(gen.HANKEL, n, P, seed=11)
        a, sa = hk.to_device(am, asg)
        x, sx = hk.to_device(xm, xsg)
        L32 = 2 * hk.limbs(P)
        y_ntt = hk.to_host(*hk.matvec(hk.HANKEL, a, sa, x, sx, P))
        y_sb = hk.to_host(*hk.schoolbook_matvec(hk.HANKEL, a, sa, x, sx, P))
        y_ka = hk.to_host(*hk.karatsuba_matvec(a, sa, x, sx, P, cutoff=args.cutoff))
        Ly = y_ntt[0].shape[1]
        agree = all(np.array_equal(y_ntt[0], y[0][:, :Ly]) and np.array_equal(y_ntt[1], y[1])
                    and not y[0][:, Ly:].any() for y in (y_sb, y_ka))
        reps = 20 if n * n * L32 * L32 < 5e10 else 5
        t_ntt = timeit(lambda: hk.matvec(hk.HANKEL, a, sa, x, sx, P), reps)
        t_sb = timeit(lambda: hk.schoolbook_matvec(hk.HANKEL, a, sa, x, sx, P), reps)
        t_ka = timeit(lambda: hk.karatsuba_matvec(a, sa, x, sx, P, cutoff=args.cutoff), reps)
        sb_prod = n * n * L32 * L32
        W32 = 2 * (hk.limbs(P) + 1)  # leaf entries: W = L + 1 two's-complement limbs
        ka_prod = karatsuba_leaf_products(n, args.cutoff) * W32 * W32
        for name, t, prod in (("A6 schoolbook", t_sb, sb_prod), ("A5 Algorithm 1", t_ka, ka_prod),
                              ("NTT path", t_ntt, None)):
            rec = {"method": name, "n": n, "P": P, "ms": round(t, 4), "agree_bitwise": bool(agree)}
            if prod is not None:
                rate = prod / (t * 1e-3)
                rec.update({"limb_products": prod, "limb_products_per_s": rate,
                            "frac_of_imad_wide_peak": round(rate / wide_peak, 4)})
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
