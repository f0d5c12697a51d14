"""Host cost of one hk_matvec_stages call (Problem.run) vs its device time, and the same step
replayed from a CUDA graph, per config: wall clock of 200 back-to-back calls (the GPU starves
when the host is slower) against the device time with the host queued ahead."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

for name in (sys.argv[1:] or ["C1", "C2", "C5C"]):
    c = gen.CONFIGS[name]
    am, asg, xm, xsg = gen.config_inputs(name)
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    prob = hk.Problem(c["kind"], a, sa, x, sx, c["P"])
    for _ in range(5):
        prob.run()
    torch.cuda.synchronize()
    N = 200
    t0 = time.perf_counter()
    for _ in range(N):
        prob.run()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / N
    torch.cuda._sleep(100_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        prob.run()
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / N
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        prob.run(stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            prob.run(stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        g.replay()
    torch.cuda.synchronize()
    gwall = (time.perf_counter() - t0) * 1e3 / N
    print(json.dumps({"config": name, "wall_ms_per_call": wall, "device_ms": dev, "graph_wall_ms": gwall}))
