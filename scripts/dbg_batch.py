import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import hkinputs as gen, oracle
import paper_1402_5287_b200 as hk
kind, n, P, batch = 0, 300, 5000, 3
am, asg, _, _ = gen.make_inputs(kind, n, P, seed=61 + n)
A = hk.PreparedMatrix(kind, *hk.to_device(am, asg), P, n, batch=batch)
xs_host = [gen.uniform(400 + v, 1, n, P) for v in range(2 * batch + 1)]
want = [oracle.matvec(kind, P, am, asg, *xs_host[v]) for v in range(2 * batch + 1)]
def bad_rows(y, w):
    gm, gs = hk.to_host(*y)
    return int(((gm != w[0]).any(axis=1) | (gs != w[1])).sum())
ys_b = A.matvec_batch([hk.to_device(xm, xsg) for xm, xsg in xs_host])
print("matvec_batch 7", [bad_rows(ys_b[v], want[v]) for v in range(7)], flush=True)
devs = [hk.to_device(*xs_host[v]) for v in range(batch)]
xm = torch.stack([d[0] for d in devs]); xsg = torch.stack([d[1] for d in devs])
for trial in range(2):
    ym, ys = A.matvec_stacked(xm, xsg)
    torch.cuda.synchronize()
    print("stacked trial", trial, [bad_rows((ym[v], ys[v]), want[v]) for v in range(batch)], flush=True)
ym1, ys1 = A.matvec_stacked(xm[:1], xsg[:1])
print("stacked 1", bad_rows((ym1[0], ys1[0]), want[0]), flush=True)
ym, ys = A.matvec_stacked(xm, xsg)
print("stacked after 1", [bad_rows((ym[v], ys[v]), want[v]) for v in range(batch)], flush=True)
