"""Dev A/B: CUDA-event stage times (K1, K2, K3) of one config for the library variant in
HK_LIB_VARIANT, without result checks (variants built with HK_K3_SKIP give wrong y on purpose).
usage: HK_LIB_VARIANT=... python scripts/stage_times.py [C3] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
c = gen.CONFIGS[name]
am, asg, xm, xsg = gen.config_inputs(name)
a, sa = hk.to_device(am, asg)
x, sx = hk.to_device(xm, xsg)
prob = hk.Problem(c["kind"], a, sa, x, sx, c["P"])
st = torch.cuda.current_stream()
stages = (hk.STAGE_SLICE_ROWS, hk.STAGE_COLUMNS, hk.STAGE_FINISH)
for _ in range(5):
    prob.run()
torch.cuda.synchronize()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
for i in range(reps):
    ev[i][0].record(st)
    for j, s in enumerate(stages):
        prob.run(s)
        ev[i][j + 1].record(st)
torch.cuda.synchronize()
ms = [sum(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(reps)) / reps for j in range(3)]
print(json.dumps({"variant": os.path.basename(os.environ.get("HK_LIB_VARIANT", "default")),
                  "config": name, "K1": round(ms[0], 4), "K2": round(ms[1], 4), "K3": round(ms[2], 4)}))
