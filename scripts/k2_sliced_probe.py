"""ncu probe: one single-GPU K2 (k2_column MODE 0) and one sliced-shard K2 (MODE 5, rank 0 of G)
at C3, for comparing their per-column cost (run under ncu -k regex:k2_column)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = gen.CONFIGS["C3"]
am, asg, xm, xsg = gen.config_inputs("C3")
a, sa = hk.to_device(am, asg)
x, sx = hk.to_device(xm, xsg)
prob = hk.Problem(c["kind"], a, sa, x, sx, c["P"])
prob.run()
ws = hk.ShardWorkspace(c["kind"], c["n"], c["P"], G)
info = ws.info
ss = torch.zeros((info["slice_buffer_words"],), dtype=torch.int32, device="cuda")
send = torch.zeros((info["buffer_words"],), dtype=torch.int32, device="cuda")
hk.shard_slice(ws, 0, a, sa, x, sx, ss)
hk.shard_columns(ws, 0, ss, send)
torch.cuda.synchronize()
print("ok")
