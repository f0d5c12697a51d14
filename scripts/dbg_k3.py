"""dev: run K1-K3 for one config with the current libhk (HK_LIB_VARIANT honoured), synchronise, report the
status and the first rows that differ from the oracle (a handful of sampled rows)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import hkinputs as gen
import oracle
import paper_1402_5287_b200 as hk

for name in sys.argv[1:]:
    c = gen.CONFIGS[name] if name in gen.CONFIGS else None
    if c is None:
        kind, n, P = (int(v) for v in name.split(","))
        am, asg, xm, xsg = gen.make_inputs(kind, n, P, 3)
    else:
        kind, n, P = c["kind"], c["n"], c["P"]
        am, asg, xm, xsg = gen.config_inputs(name)
    try:
        a, sa = hk.to_device(am, asg)
        x, sx = hk.to_device(xm, xsg)
        ym, ys = hk.matvec(kind, a, sa, x, sx, P)
        torch.cuda.synchronize()
        ym, ys = hk.to_host(ym, ys)
        rows = np.unique(np.linspace(0, n - 1, min(n, 12)).astype(int))
        wm, ws = oracle.matvec(kind, P, am, asg, xm, xsg, rows=rows) if "rows" in oracle.matvec.__code__.co_varnames else oracle.matvec(kind, P, am, asg, xm, xsg)
        if wm.shape[0] != rows.size:
            wm, ws = wm[rows], ws[rows]
        bad = [int(r) for i, r in enumerate(rows) if (ym[r] != wm[i]).any() or ys[r] != ws[i]]
        print(name, "plan", {k: hk.plan(kind, n, P)[k] for k in ("w", "Ly", "log_n2")}, "bad rows", bad, flush=True)
    except Exception as e:
        print(name, "ERROR", repr(e), flush=True)
        break
