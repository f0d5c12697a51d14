"""e2e throughput (pinned host buffers -> HostPipeline -> host y) at C3 vs pipeline depth, beside the
box's pinned copy rates; shows whether the end-to-end number is copy-engine / PCIe bound."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

kind, n, P = 0, 8000, 33216
am, asg, xm, xsg = gen.config_inputs("C3")
pa, ps = torch.from_numpy(am.view("int64")).pin_memory(), torch.from_numpy(asg).pin_memory()
px, pxs = torch.from_numpy(xm.view("int64")).pin_memory(), torch.from_numpy(xsg).pin_memory()
Ly = hk.out_limbs(P)
h2d = am.nbytes + xm.nbytes
d2h = n * Ly * 8
dev = torch.empty(h2d // 8 + 1, dtype=torch.int64, device="cuda")
hb = torch.empty(h2d // 8 + 1, dtype=torch.int64).pin_memory()
for _ in range(3):
    dev.copy_(hb, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    dev.copy_(hb, non_blocking=True)
torch.cuda.synchronize()
print({"h2d_GBps": 10 * hb.nbytes / (time.perf_counter() - t0) / 1e9})
for depth in (2, 3, 4, 6):
    pipe = hk.HostPipeline(kind, n, P, depth=depth)
    outs = [(torch.empty((n, Ly), dtype=torch.int64).pin_memory(),
             torch.empty((n,), dtype=torch.int8).pin_memory()) for _ in range(depth)]
    for i in range(2 * depth):
        pipe.submit(pa, ps, px, pxs, outs[i % depth])
    pipe.drain()
    K = 30
    t0 = time.perf_counter()
    for i in range(K):
        pipe.submit(pa, ps, px, pxs, outs[i % depth])
    pipe.drain()
    ms = (time.perf_counter() - t0) * 1e3 / K
    print({"depth": depth, "ms_per_matvec": round(ms, 3), "matvec_per_s": round(1000 / ms, 1),
           "h2d_GBps_effective": round(h2d / ms / 1e6, 1), "bound_ms_h2d_55GBps": round(h2d / 55e6, 3)})
    del pipe, outs
    torch.cuda.empty_cache()
