"""Per-rank compute time of the sigma-coset shards (SURVEY 8(e) plan P-2) measured on ONE B200 by
running one rank's kernels alone (no other rank, no exchange): hk_hankel_shard_forward (K1 with the
coset fold + K2 on N2/G columns) and hk_hankel_shard_finish (K3 on n/G rows), CUDA events, C3 by
default.  Compute-only scaling efficiency E_G = T_1 / (G T_G), T_G = max over the ranks timed.
Sliced sharding (hk_hankel_shard_slice / _columns / _finish): every rank timed; the slice and coset
exchange volumes per rank are reported in bytes (at NVLink 5's 900 GB/s per direction they add
bytes / 900e9 s when not overlapped)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hkinputs as gen  # noqa: E402
import paper_1402_5287_b200 as hk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = 20
c = gen.CONFIGS[name]
kind, n, P = c["kind"], c["n"], c["P"]
am, asg, xm, xsg = gen.config_inputs(name)
a, sa = hk.to_device(am, asg)
x, sx = hk.to_device(xm, xsg)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


prob = hk.Problem(kind, a, sa, x, sx, P)
t1 = timed(prob.run)
res = {"config": name, "T1_ms": t1, "ranks": {}}
for G in (2, 4, 8):
    ws = hk.ShardWorkspace(kind, n, P, G)
    info = ws.info
    send = torch.zeros((info["buffer_words"],), dtype=torch.int32, device="cuda")
    yr, Ly = info["y_rows"], hk.out_limbs(P)
    ym = torch.zeros((yr, Ly), dtype=torch.int64, device="cuda")
    ys = torch.zeros((yr,), dtype=torch.int8, device="cuda")
    worst = 0.0
    per = {}
    for g in sorted({0, G - 1}):
        tf = timed(lambda: hk.shard_forward(ws, g, a, sa, x, sx, send))
        tk = timed(lambda: hk.shard_finish(ws, g, send, ym, ys))  # send stands in for the receive buffer
        per[g] = {"forward_K1K2_ms": tf, "finish_K3_ms": tk}
        worst = max(worst, tf + tk)
    res["ranks"][G] = {"per_rank": per, "T_G_ms": worst, "E_compute": t1 / (G * worst)}
    if info["slice_buffer_words"]:
        ssend = torch.zeros((info["slice_buffer_words"],), dtype=torch.int32, device="cuda")
        sper, sworst = {}, 0.0
        for g in range(G):
            ts = timed(lambda: hk.shard_slice(ws, g, a, sa, x, sx, ssend))
            tc = timed(lambda: hk.shard_columns(ws, g, ssend, send))
            tk = per[min(per, key=lambda r: abs(r - g))]["finish_K3_ms"]
            sper[g] = {"slice_K1_ms": ts, "columns_K2_ms": tc, "finish_K3_ms": tk}
            sworst = max(sworst, ts + tc + tk)
        sb = 4 * info["slice_chunk_words"] * (G - 1)
        cb = 4 * info["chunk_words"] * (G - 1)
        res["ranks"][G]["sliced"] = {
            "per_rank": sper, "T_G_ms": sworst, "E_compute": t1 / (G * sworst),
            "slice_exchange_bytes_per_rank": sb, "coset_exchange_bytes_per_rank": cb,
            "exchange_ms_at_900GBs": (sb + cb) / 900e9 * 1e3}
        del ssend
    del ws, send, ym, ys
print(json.dumps(res, indent=1))
