"""Device time of one call (no host launch overhead): a GPU sleep first lets the host queue
`reps` calls, which then run back to back between two CUDA events.
usage: python scripts/device_time.py [cases n:P,...]   (A6 schoolbook, A5 Algorithm 1, NTT path)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

cases = [tuple(map(int, c.split(":"))) for c in (sys.argv[1] if len(sys.argv) > 1 else "64:3328").split(",")]


def dev_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)  # ~25 ms of GPU time to queue behind
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n, P in cases:
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=1)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    Ly = hk.out_limbs(P)
    out = (torch.empty((n, Ly), dtype=torch.int64, device="cuda"), torch.empty((n,), dtype=torch.int8, device="cuda"))
    prob = hk.Problem(0, a, sa, x, sx, P)
    r = {"n": n, "P": P,
         "A6_schoolbook_ms": dev_ms(lambda: hk.schoolbook_matvec(0, a, sa, x, sx, P, out=out)),
         "ntt_path_ms": dev_ms(prob.run)}
    print(json.dumps(r))
