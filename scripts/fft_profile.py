"""F3 (hk_fft_matvec) at a BASELINE config: one warm-up call and a few timed calls, for ncu launch
lists / captures of the FP64 FFT kernels (scripts/gpu_fft_profile.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = gen.CONFIGS[name]
am, asg, xm, xsg = gen.config_inputs(name)
a, sa = hk.to_device(am, asg)
x, sx = hk.to_device(xm, xsg)
ws = hk.FftWorkspace(c["kind"], c["n"], c["P"])
out = hk.fft_matvec(c["kind"], a, sa, x, sx, c["P"], ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    hk.fft_matvec(c["kind"], a, sa, x, sx, c["P"], out=out, ws=ws, check=False)
e1.record()
torch.cuda.synchronize()
print(name, hk.fft_plan(c["kind"], c["n"], c["P"]), "ms per matvec", e0.elapsed_time(e1) / reps)
