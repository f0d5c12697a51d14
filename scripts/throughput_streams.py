"""Device-resident throughput with S independent C3 problems in flight on S streams (kernel tails of
one problem overlap the next problem's kernels).  Secondary measurement; bench.py's value is one
matvec per step."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = 60
kind, n, P = 0, 8000, 33216
probs, streams = [], []
for s in range(S):
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=2 + s)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    probs.append(hk.Problem(kind, a, sa, x, sx, P))
    streams.append(torch.cuda.Stream())
torch.cuda.synchronize()
for it in range(3):
    for s in range(S):
        probs[s].run(stream=streams[s])
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(K):
    for s in range(S):
        probs[s].run(stream=streams[s])
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / (K * S)
print(f"S={S}: {dt * 1e3:.3f} ms per matvec, {1 / dt:.1f} matvec/s")
