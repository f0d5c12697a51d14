import faulthandler, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.enable()
import numpy as np, torch
import hkinputs as gen, oracle
import paper_1402_5287_b200 as hk
am, asg, xm, xsg = gen.make_inputs(0, 64, 3328, 0)
print("A", flush=True)
ws = hk.FftWorkspace(0, 64, 3328)
print("B ws", ws.nbytes, flush=True)
torch.cuda.synchronize()
print("C", ws.status(), flush=True)
a, sa = hk.to_device(am, asg); x, sx = hk.to_device(xm, xsg)
ym, ys = hk.fft_matvec(0, a, sa, x, sx, 3328, ws=ws, check=False)
print("D", flush=True)
torch.cuda.synchronize()
print("E", ws.status(), flush=True)
gm, gs = hk.to_host(ym, ys)
wm, ws_ = oracle.matvec(0, 3328, am, asg, xm, xsg)
print("rows differ", int(((gm != wm).any(axis=1) | (gs != ws_)).sum()), flush=True)
