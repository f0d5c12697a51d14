#!/usr/bin/env python
"""F2: crossover sweep on B200 of the three GPU methods for the exact Hankel
matvec at P = 33,216 bits -- the 2-D NTT path (hk_hankel_matvec), the direct schoolbook limb
kernel (A6, hk_schoolbook_matvec) and the paper's Algorithm 1 level by level (A5,
hk_karatsuba_matvec) -- mirroring the paper's only empirical statement ("for b = 32768 bits
accuracy, FFT becomes superior only for n > 8000") on this hardware.

Times are device times per call on resident inputs (CUDA events around calls queued behind a
GPU sleep); a method is skipped once a single call is
predicted to exceed --budget seconds.  Results agree bit for bit between methods (checked for
every n measured).  Prints one JSON line per (method, n) and a markdown table.
"""
import argparse
import json
import os
import statistics  # noqa: F401
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402


def timeit(fn, reps):
    """Device time per call: the calls are queued behind a GPU sleep, so host launch work (which
    bounds single small calls) is not in the events."""
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    one = time.perf_counter() - t0
    reps = max(1, min(reps, int(0.3 / max(one, 1e-6))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(min(2e9, 4e5 * reps)))
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=33216)
    ap.add_argument("--budget", type=float, default=1.5)
    ap.add_argument("--max-n", type=int, default=16384)
    ap.add_argument("--cutoff", type=int, default=8)
    args = ap.parse_args()
    P = args.P
    ns = [n for n in [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8000, 8192, 16384]
          if n <= args.max_n]
    rows = []
    last = {}
    for n in ns:
        am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=n)
        a, sa = hk.to_device(am, asg)
        x, sx = hk.to_device(xm, xsg)
        res = {}
        # NTT path (resident workspace, stage API = the same 5 launches as hk_hankel_matvec)
        prob = hk.Problem(0, a, sa, x, sx, P)
        ms = timeit(prob.run, 20)
        res["ntt"] = ms
        ref = hk.to_host(prob.y_mag, prob.y_sign)
        for meth in ("schoolbook", "karatsuba"):
            pred = last.get(meth)
            if pred is not None and pred[1] * (n / pred[0]) ** (2.0 if meth == "schoolbook" else 1.6) > args.budget * 1e3:
                continue
            if meth == "karatsuba" and hk.karatsuba_workspace_size(n, P, args.cutoff) > 60e9:
                continue
            if meth == "schoolbook":
                fn = lambda: hk.schoolbook_matvec(0, a, sa, x, sx, P)  # noqa: E731
            else:
                fn = lambda: hk.karatsuba_matvec(a, sa, x, sx, P, cutoff=args.cutoff)  # noqa: E731
            out = fn()
            torch.cuda.synchronize()
            got = hk.to_host(*out)
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), (meth, n)
            ms = timeit(fn, 5)
            res[meth] = ms
            last[meth] = (n, ms)
        for meth, ms in res.items():
            line = {"method": meth, "n": n, "P": P, "ms": ms, "matvec_per_s": 1e3 / ms}
            print(json.dumps(line), flush=True)
        rows.append((n, res))
        del prob
        torch.cuda.empty_cache()
    print("\n| n | NTT path (ms) | schoolbook A6 (ms) | Algorithm 1 A5 (ms) | fastest |")
    print("|---|---|---|---|---|")
    for n, res in rows:
        best = min(res, key=res.get)
        f = lambda k: f"{res[k]:.3f}" if k in res else "—"  # noqa: E731
        print(f"| {n} | {f('ntt')} | {f('schoolbook')} | {f('karatsuba')} | {best} |")


if __name__ == "__main__":
    main()
