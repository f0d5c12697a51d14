import sys, numpy as np, torch
sys.path.insert(0, '.')
import hkinputs as gen, paper_1402_5287_b200 as hk
n, P = int(sys.argv[1]), int(sys.argv[2])
am, asg, xm, xsg = gen.make_inputs(0, n, P, 0)
ym, ys = hk.hankel_matvec(*hk.to_device(am, asg), *hk.to_device(xm, xsg), P)
torch.cuda.synchronize(); print("ok", n, P)
