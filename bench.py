#!/usr/bin/env python
"""bench.py -- exact multiprecision Hankel matvec throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {hk,reference}] [--config C3]

A step is one full matvec (all SURVEY.md 8(a) rows A1-A4: slicing, 2-D forward NTT, pointwise,
inverse NTT, CRT, carry) over the BASELINE workload, with inputs resident in HBM.  N = 1 runs
C3 (Hankel n = 8000, P = 33,216 bits, seed 2).  N > 1 (torchrun, NCCL) runs the row-block plan
of paper_1402_5287_b200.dist: each rank computes its nr x n Hankel window with the CUDA path and
the y rows are all-gathered; value = matvecs/s of the whole job, time = max over ranks.

--impl reference times the oracle (plain C schoolbook, oracle/) on the host cores on a bounded
sample of output rows of the same workload (all rows cost the same n L^2 limb products).
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hkinputs as gen  # noqa: E402

METRIC = "Hankel matvecs/sec at n=8000, P=33,216 bits"
UNIT = "matvec/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT_B200 = 148
LANES_PER_SM = 128  # 4 SMSPs x 32 lanes: issue limit of integer instructions per clock
# algorithmic SASS instructions per operation of the number system
I_GS, I_CT, I_MONT = 7, 8, 4
# Integer-pipe roofline: per SMSP the FMA pipe takes IMAD every 2 clocks and
# IMAD.HI / IMAD.WIDE every 4 (scripts/micro_pipes.cu), the ALU pipe every 2.  Minimal pipe clocks
# per warp-operation: GS butterfly 8 (IMAD.HI + 2 IMAD; its 4 ALU ops fit beside them), CT
# butterfly 9 (8 FMA + 10 ALU, balanced by moving one add onto the FMA pipe), Montgomery product
# 10 (2 IMAD.WIDE + IMAD).  Peak = 4 SMSPs x 32 lanes / 8 clocks = 16 GS butterflies/clk/SM.
C_GS, C_CT, C_MONT = 8, 9, 10
BFLY_PER_CLK_SM = 16
# measured register-resident ceilings (scripts/micro_bfly.cu, profiles/r01/micro_bfly.log)
MICRO_GS, MICRO_CT = 12.07, 11.22  # butterflies / clk / SM
# SURVEY.md 8(d) roofline: I_alg = 8 butterflies + 6 pointwise + 15 slice-residues + C_CRT CRT
# coefficients + C_CARRY carry limbs, against 128 thread-instructions / clk / SM.  The survey's
# CRT / carry constants (110 / 25) were estimates; C_CRT and C_CARRY are the counts of the
# current K3's SASS (scripts/k3_sass_counts.py): SASS instructions per
# Garner coefficient of the CRT loop and per output limb of the carry phase.
S_BFLY, S_PW, S_RES = 8, 6, 15
S_CRT_SURVEY, S_CARRY_SURVEY = 110, 25
C_CRT, C_CARRY = 112, 75  # profiles/r02/k3_sass_counts.json (k3_finish<10,13>)


def survey_model(plan, m=None):
    """SURVEY.md 8(d) algorithmic instruction counts per matvec, split by kernel (full
    transforms, no pruning credit)."""
    k = plan["k_primes"]
    N1, N2 = 1 << plan["log_n1"], 1 << plan["log_n2"]
    lg1, lg2 = plan["log_n1"], plan["log_n2"]
    rows_a, n = plan["a_count"], plan["n"]
    m = plan["m"] if m is None else m
    bf_k1 = k * (rows_a + n) * (N2 // 2) * lg2
    bf_k2 = 3 * k * N2 * (N1 // 2) * lg1
    bf_k3 = k * m * (N2 // 2) * lg2
    pointwise = k * N2 * N1
    residues = k * (rows_a + n) * plan["Ls"]
    crt = m * (2 * plan["Ls"] - 1)
    limbs = m * plan["Ly"]
    i_k1 = S_BFLY * bf_k1 + S_RES * residues
    i_k2 = S_BFLY * bf_k2 + S_PW * pointwise
    i_k3 = S_BFLY * bf_k3 + C_CRT * crt + C_CARRY * limbs
    i_k3_survey = S_BFLY * bf_k3 + S_CRT_SURVEY * crt + S_CARRY_SURVEY * limbs
    return dict(butterflies=bf_k1 + bf_k2 + bf_k3, pointwise=pointwise, residues=residues, crt=crt,
                carry_limbs=limbs, K1=i_k1, K2=i_k2, K3=i_k3, K3_survey_constants=i_k3_survey,
                total=i_k1 + i_k2 + i_k3)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hk", choices=["hk", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(gen.CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N = 1: launch every timed step from the host instead of replaying its CUDA graph")
    ap.add_argument("--plan", default="coset", choices=["coset", "rowblock"],
                    help="multi-GPU plan (N > 1): SURVEY 8(e) P-2 sigma-coset (default) or P-3 row blocks")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
def workload(cfg_name):
    c = gen.CONFIGS[cfg_name]
    kind = c["kind"]
    return dict(name=cfg_name, kind=kind, n=c["n"], P=c["P"], seed=c["seed"], recipe=c["recipe"],
                desc=f"{cfg_name} {gen.KIND_NAMES[kind]} n={c['n']} P={c['P']} seed={c['seed']} "
                     f"{c['recipe']}")


def pcie_roofline(h2d, d2h, ms_e2e, dev):
    """The e2e step's own roofline: pinned-copy bandwidth of this box measured here (64 MiB copies,
    CUDA events; H2D and D2H concurrently on two streams, as the pipeline runs them), and the
    fraction of the e2e step those bytes need at that rate."""
    import torch
    nb = 64 << 20
    hs = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
    ds = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def both():
        with torch.cuda.stream(s1):
            ds[0].copy_(hs[0], non_blocking=True)
        with torch.cuda.stream(s2):
            hs[1].copy_(ds[1], non_blocking=True)

    def one(up):
        with torch.cuda.stream(s1):
            (ds[0].copy_(hs[0], non_blocking=True) if up else hs[1].copy_(ds[1], non_blocking=True))

    res = {}
    for name, fn in (("h2d", lambda: one(True)), ("d2h", lambda: one(False)), ("both", both)):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        res[name] = (2 if name == "both" else 1) * 5 * nb / (time.perf_counter() - t0) / 1e9
    t_copy = max(h2d / (res["h2d"] * 1e9), d2h / (res["d2h"] * 1e9), (h2d + d2h) / (res["both"] * 1e9))
    return {"h2d_gbs": res["h2d"], "d2h_gbs": res["d2h"], "bidir_gbs": res["both"],
            "t_copy_ms": t_copy * 1e3, "frac": t_copy * 1e3 / ms_e2e,
            "what": "pinned host<->device bandwidth measured in this run (64 MiB copies, wall clock); "
                    "t_copy = max(h2d / H2D, d2h / D2H, (h2d + d2h) / bidirectional); frac = t_copy / e2e step"}


def workload_config(wl):
    """The `config` object, identical for both arms (the workload, and the L2 note the contract asks for)."""
    return {"workload": wl["desc"], "kind": gen.KIND_NAMES[wl["kind"]], "n": wl["n"], "P": wl["P"],
            "l2": "no flush: every step streams its own inputs and transform-domain arrays (C3: 100 MB of "
                  "inputs + 1.48 GB of transform-domain traffic), far beyond the 126 MB L2"}


def alg_counts(plan, m=None):
    """Algorithmic operation counts per matvec: full transforms, no
    pruning credit."""
    k = plan["k_primes"]
    N1, N2 = 1 << plan["log_n1"], 1 << plan["log_n2"]
    lg1, lg2 = plan["log_n1"], plan["log_n2"]
    rows_a, n = plan["a_count"], plan["n"]
    m = plan["m"] if m is None else m
    bf_row_fwd = k * (rows_a + n) * (N2 // 2) * lg2
    bf_col_fwd = k * N2 * 2 * (N1 // 2) * lg1
    bf_col_inv = k * N2 * (N1 // 2) * lg1
    bf_row_inv = k * m * (N2 // 2) * lg2
    pointwise = k * N2 * N1
    k2_instr = I_GS * bf_col_fwd + I_CT * bf_col_inv + I_MONT * pointwise
    k2_bfly_eq = (C_GS * bf_col_fwd + C_CT * bf_col_inv + C_MONT * pointwise) / C_GS
    # K1: slice NTTs of a and x (GS) + 2 Shoup products per slice residue; K3: inverse slice NTTs
    # (CT) + Garner CRT per output coefficient (10 Shoup products = 80 FMA clocks + ~10 IMAD.WIDE
    # = 40 -> 120 clocks = 15 GS-eq); carries are ALU work and not counted
    residues = k * (rows_a + n) * plan["Ls"]
    k1_bfly_eq = bf_row_fwd + 2 * residues
    k3_bfly_eq = (C_CT * bf_row_inv) / C_GS + 15 * m * (2 * plan["Ls"] - 1)
    return dict(bf_row_fwd=bf_row_fwd, bf_col_fwd=bf_col_fwd, bf_col_inv=bf_col_inv,
                bf_row_inv=bf_row_inv, pointwise=pointwise, k2_instr=k2_instr,
                k2_bfly_eq=k2_bfly_eq, k1_bfly_eq=k1_bfly_eq, k3_bfly_eq=k3_bfly_eq,
                butterflies=bf_row_fwd + bf_col_fwd + bf_col_inv + bf_row_inv)


def alg_bytes(plan):
    """Algorithmic HBM bytes per matvec: a, x, y once + one write and one read of each
    transform-domain array (A^, X^ row pass outputs, Y^ column pass output)."""
    L, Ly, k = plan["L"], plan["Ly"], plan["k_primes"]
    N2 = 1 << plan["log_n2"]
    io = (plan["a_count"] + plan["n"]) * (8 * L + 1) + plan["m"] * (8 * Ly + 1)
    inter = 2 * 4 * k * N2 * (plan["a_count"] + plan["n"] + plan["m"])
    return io, io + inter


def verify_y(kind, am, asg, xm, xsg, y_mag, y_sign, rank, world, dist, dev):
    """Check of the whole first y before timing: Y mod q of every row against the inputs mod q
    for three primes q < 2^24 (tests/fingerprint.py: reduction mod q is a ring homomorphism, so it
    holds at any size).  Rank 0 checks; the verdict is shared with every rank."""
    ok, why = True, None
    if rank == 0:
        from tests import fingerprint as fp
        ym = y_mag.cpu().numpy().view(np.uint64)
        ys = y_sign.cpu().numpy()
        try:
            fp.check(kind, am, asg, xm, xsg, ym, ys)
        except AssertionError as e:
            ok, why = False, str(e)[:200]
    if world > 1:
        import torch
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = bool(t.item())
    return ok, why


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = []
        for ts, line in self.samples:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((ts, float(parts[0]), float(parts[1]), parts[3:]))
            except ValueError:
                continue
        inside = [r for r in rows if t0 - 0.05 <= r[0] <= t1 + 0.05]
        use = inside if inside else rows[-5:]
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in use for i, v in enumerate(r[3]) if v.startswith("Active")})
        return {"sm_mhz": statistics.median(r[1] for r in use), "sm_max_mhz": max(r[2] for r in use),
                "reasons": reasons, "samples": len(use), "in_timed_region": bool(inside)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, min_rows=64, y_gpu=None):
    """The oracle as it stands, on a bounded sample of output rows (>= 64, a multiple of the core
    count), all host cores.  With ``y_gpu`` (host copies of the GPU's y) the sampled
    rows are also compared with the GPU's, limb for limb."""
    import oracle
    kind, n, P = wl["kind"], wl["n"], wl["P"]
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, wl["seed"], wl["recipe"])
    cores = oracle.default_threads()
    R = min(n, -(-min_rows // cores) * cores)
    rows = np.linspace(0, n - 1, R).astype(np.int64)
    t0 = time.perf_counter()
    wm, ws_ = oracle.matvec(kind, P, am, asg, xm, xsg, rows=rows, threads=cores)
    dt = time.perf_counter() - t0
    out = {"value": (R / n) / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"{R} of {n} output rows of {wl['name']} (evenly spaced; each row = n*L^2 = "
                     f"{n * gen.n_limbs(P) ** 2:.3g} limb products), {dt:.2f} s on {cores} threads, "
                     f"extrapolated to whole matvecs"}
    if y_gpu is not None:
        gm, gs = y_gpu
        bad = int(((gm[rows] != wm).any(axis=1) | (gs[rows] != ws_)).sum())
        out["gpu_rows_checked"] = R
        out["gpu_rows_differing"] = bad
    return out


# ---------------------------------------------------------------------------------------------
def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build_oracle()
    vals = []
    t_all = time.perf_counter()
    cb = None
    budget_s = float(os.environ.get("HK_REFERENCE_BUDGET_S", "240"))
    steps_run = 0
    for _ in range(args.steps):  # each step: one row per host thread (bounded sample)
        cb = cpu_baseline(wl)
        vals.append(cb["value"])
        steps_run += 1
        if time.perf_counter() - t_all > budget_s:
            break
    value = statistics.median(vals)
    ms = 1000.0 / value
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps_run, "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(wl),
            "cpu_baseline": {**cb, "value": value},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    wl = workload(args.config)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1402_5287_b200 as hk

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    kind, n, P = wl["kind"], wl["n"], wl["P"]
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, wl["seed"], wl["recipe"])
    a, sa = hk.to_device(am, asg, dev)
    x, sx = hk.to_device(xm, xsg, dev)
    stream = torch.cuda.current_stream()

    plan = hk.plan(kind, n, P)
    W, K = max(3, args.warmup), args.steps
    sh_verified_p2p = False
    stage_names = ("K1_slice_rowntt", "K2_column", "K3_finish")
    if world == 1:
        prob = hk.Problem(kind, a, sa, x, sx, P)
        prob.run()
        if prob.status() != hk.HK_OK:
            raise SystemExit("bench: device status not OK")
        ok, why = verify_y(kind, am, asg, xm, xsg, prob.y_mag, prob.y_sign, 0, 1, None, dev)
        verification = {"fingerprints_all_rows": ok, "detail": why}
        if not ok:
            raise SystemExit(f"bench: y fails its fingerprints ({why})")
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]

        if not args.no_graph:  # whole steps replayed from a CUDA graph (one host call per step)
            prob.capture()

        def step(i=None):
            if i is None:
                prob.run() if args.no_graph else prob.replay()
                return
            e = ev[i]
            e[0].record(stream)
            prob.run(hk.STAGE_SLICE_ROWS)
            e[1].record(stream)
            prob.run(hk.STAGE_COLUMNS)
            e[2].record(stream)
            prob.run(hk.STAGE_FINISH)
            e[3].record(stream)
        launches_per_step = 3  # K1 (a and x tiles), K2, K3
    elif args.plan == "coset":
        # SURVEY 8(e) plan P-2: coset-sharded K1/K2 -> NCCL all-to-all -> row-block K3 ->
        # NCCL all-gather of y; stages: forward, all-to-all, finish + all-gather
        from paper_1402_5287_b200 import dist as hkdist
        sh = hkdist.CosetShardedMatvec(kind, a, sa, x, sx, P)
        sh.step(check=True)
        ok, why = verify_y(kind, am, asg, xm, xsg, *sh.result(), rank, world, dist, dev)
        verification = {"fingerprints_all_rows": ok, "p2p_tried": sh.p2p, "sliced_tried": sh.sliced,
                        "detail": why}
        # a wrong y (all ranks agree: verify_y all-reduces) falls back one mechanism at a time:
        # NCCL exchanges instead of peer memory, then the coset (unsliced) forward phase
        for kw, what in (({"p2p": False}, "NCCL exchanges"), ({"p2p": False, "sliced": False},
                                                              "NCCL exchanges, unsliced forward")):
            if ok or (not sh.p2p and not sh.sliced):
                break
            if "sliced" not in kw and not sh.p2p:
                continue
            sh = hkdist.CosetShardedMatvec(kind, a, sa, x, sx, P, **kw)
            sh.step(check=True)
            ok, why = verify_y(kind, am, asg, xm, xsg, *sh.result(), rank, world, dist, dev)
            verification.update(fingerprints_all_rows=ok, fallback=what + " after a mismatch", detail=why)
        if not ok:
            raise SystemExit(f"bench: sharded y fails its fingerprints ({why})")
        sh_verified_p2p = sh.p2p
        if sh.sliced:
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(K)]
            stage_names = ("shard_slice_K1", "slice_all_to_all", "shard_columns_K2", "all_to_all",
                           "shard_finish_K3+all_gather")
        else:
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
            stage_names = ("shard_forward_K1K2", "all_to_all", "shard_finish_K3+all_gather")

        def step(i=None):
            if i is None:
                sh.step()
                return
            e = ev[i]
            e[0].record(stream)
            if sh.sliced:
                sh.compute_slice()
                e[1].record(stream)
                sh.exchange_slices()
                e[2].record(stream)
                sh.compute_columns()
                e = e[2:]
            else:
                sh.compute_forward()
            e[1].record(stream)
            sh.exchange()
            e[2].record(stream)
            sh.compute_finish()
            sh.gather()
            e[3].record(stream)
        # coset: K1 (coset block), K2 (N2/G columns), K3 (row block); sliced: K1 runs as two
        # launches (this rank's a positions, its x positions)
        launches_per_step = 4 if sh.sliced else 3
    else:
        from paper_1402_5287_b200 import dist as hkdist
        sh = hkdist.ShardedHankel(a, sa, x, sx, P)
        sh.step(check=True)
        ok, why = verify_y(kind, am, asg, xm, xsg, *sh.result(), rank, world, dist, dev)
        verification = {"fingerprints_all_rows": ok, "detail": why}
        if not ok:
            raise SystemExit(f"bench: row-block y fails its fingerprints ({why})")
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
        stage_names = ("-", "shard_compute", "all_gather")

        def step(i=None):
            if i is None:
                sh.step()
                return
            e = ev[i]
            e[0].record(stream)
            e[1].record(stream)
            if sh.nr > 0:
                sh.compute(sh.win[0], sh.win[1], sh.x[0], sh.x[1], P, sh.nr,
                           out=(sh.y_loc[: sh.nr], sh.s_loc[: sh.nr]), ws=sh.ws)
            e[2].record(stream)
            sh._gather()
            e[3].record(stream)
        launches_per_step = 3  # K1, K2, K3 of the row-block shard

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        time.sleep(0.3)
    # ---- timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    # single GPU: the timed steps are whole matvecs (one hk_matvec_stages call each); the per-stage
    # times come from a separate pass below (per-stage calls add host work that small configs feel)
    stages_apart = world == 1
    t_start.record(stream)
    for i in range(K):
        step(None if stages_apart else i)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall1 = time.time()
    ms_total = t_start.elapsed_time(t_end)
    if world > 1:
        tt = torch.tensor([ms_total], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / K
    if stages_apart:  # stage pass: queued behind a GPU sleep so the events see device time only
        torch.cuda._sleep(int(2e6 + 2e5 * K))
        for i in range(K):
            step(i)
        torch.cuda.synchronize()
    stage_ms = [statistics.mean(ev[i][s].elapsed_time(ev[i][s + 1]) for i in range(K))
                for s in range(len(stage_names))]
    clocks = sampler.summary(wall0, wall1) if sampler else None
    if sampler:
        sampler.stop()

    # ---- F1 (secondary): fixed A, new x each step (prepared 2-D transform of a)
    warm = None
    if rank == 0 and world == 1:
        A = hk.PreparedMatrix(kind, a, sa, P, n)
        yb = (torch.empty((n, plan["Ly"]), dtype=torch.int64, device=dev),
              torch.empty((n,), dtype=torch.int8, device=dev))
        for _ in range(W):
            A.matvec(x, sx, out=yb, check=False)
        torch.cuda.synchronize()
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        for _ in range(K):
            A.matvec(x, sx, out=yb, check=False)
        w1.record(stream)
        torch.cuda.synchronize()
        if A.ws.status() != hk.HK_OK:
            raise SystemExit("bench: prepared-matvec status not OK")
        wms = w0.elapsed_time(w1) / K
        warm = {"value": 1000.0 / wms, "unit": UNIT, "ms_per_step": wms,
                "what": "same matvec with the 2-D transform of a prepared once (hk_prepare_a); "
                        "per step: x slicing + transforms, pointwise, inverse, CRT, carry"}
        del A
        # F1 multi-vector batching: 3 lanes (streams with their own prepared copy), 3 vectors per round
        LN = 3
        A = hk.PreparedMatrix(kind, a, sa, P, n, lanes=LN)
        outs = [(torch.empty((n, plan["Ly"]), dtype=torch.int64, device=dev),
                 torch.empty((n,), dtype=torch.int8, device=dev)) for _ in range(LN)]
        for _ in range(W):
            A.matvec_batch([(x, sx)] * LN, outs=outs, check=False)
        torch.cuda.synchronize()
        w0.record(stream)
        for _ in range(K):
            A.matvec_batch([(x, sx)] * LN, outs=outs, check=False)
        w1.record(stream)
        torch.cuda.synchronize()
        for lw in A._lane_ws:
            if lw.status() != hk.HK_OK:
                raise SystemExit("bench: batched prepared-matvec status not OK")
        bms = w0.elapsed_time(w1) / (K * LN)
        warm["batch"] = {"value": 1000.0 / bms, "unit": UNIT, "ms_per_matvec": bms, "lanes": LN,
                         "what": "PreparedMatrix.matvec_batch: 3 vectors per call over 3 lanes "
                                 "(CUDA streams, each with its own prepared copy of a's transform); "
                                 "CUDA events on the calling stream, which waits for every lane"}
        del A, outs
        # F1 kernel-level batch: one prepared copy of a's transform, 4 vectors per launch of each kernel
        KB_ = 4
        A = hk.PreparedMatrix(kind, a, sa, P, n, batch=KB_)
        xb_m = x.unsqueeze(0).expand(KB_, -1, -1).contiguous()
        xb_s = sx.unsqueeze(0).expand(KB_, -1).contiguous()
        yb4 = (torch.empty((KB_, n, plan["Ly"]), dtype=torch.int64, device=dev),
               torch.empty((KB_, n), dtype=torch.int8, device=dev))
        for _ in range(W):
            A.matvec_stacked(xb_m, xb_s, out=yb4, check=False)
        torch.cuda.synchronize()
        w0.record(stream)
        for _ in range(K):
            A.matvec_stacked(xb_m, xb_s, out=yb4, check=False)
        w1.record(stream)
        torch.cuda.synchronize()
        if A.ws.status() != hk.HK_OK:
            raise SystemExit("bench: kernel-batched prepared-matvec status not OK")
        kbms = w0.elapsed_time(w1) / (K * KB_)
        warm["kernel_batch"] = {"value": 1000.0 / kbms, "unit": UNIT, "ms_per_matvec": kbms, "vectors_per_launch": KB_,
                                "what": "PreparedMatrix(batch=4).matvec_stacked -> hk_matvec_prepared_batch: one launch "
                                        "of K1 / K2 / K3 for 4 vectors, one prepared copy of a's transform (each A^ "
                                        "column read from HBM once per batch)"}
        del A, xb_m, xb_s, yb4

    # ---- throughput mode: a stream of >= 16 independent matvecs with several
    # in flight; at N = 1 three Problems (own workspaces and y) on three streams, at N > 1 the
    # sigma-coset CosetStream (3 slots, exchanges on a communication stream).  T = device time of
    # the whole stream / count (CUDA events on the calling stream, which joins every stream), max
    # over ranks; the latency-mode headline (one matvec per step) is kept as `value`.
    throughput = None
    n_tp = max(16, min(K, 64))
    if world == 1:
        S_ = 3
        others = [prob]
        for sidx in range(1, S_):
            am2, asg2, xm2, xsg2 = gen.make_inputs(kind, n, P, wl["seed"] + 100 * sidx, wl["recipe"])
            a2, sa2 = hk.to_device(am2, asg2, dev)
            x2, sx2 = hk.to_device(xm2, xsg2, dev)
            others.append(hk.Problem(kind, a2, sa2, x2, sx2, P))
        strs = [torch.cuda.Stream(device=dev) for _ in range(S_)]

        def tp_round(count):
            for st in strs:
                st.wait_stream(stream)
            for t in range(count):
                others[t % S_].run(stream=strs[t % S_])
            for st in strs:
                stream.wait_stream(st)

        tp_round(2 * S_)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        tp_round(n_tp)
        c1.record(stream)
        torch.cuda.synchronize()
        cms = c0.elapsed_time(c1) / n_tp
        for pr in others:
            if pr.status() != hk.HK_OK:
                raise SystemExit("bench: throughput-mode status not OK")
        throughput = {"value": 1000.0 / cms, "unit": UNIT, "ms_per_matvec": cms, "matvecs": n_tp,
                      "in_flight": S_, "launches": 3 * n_tp,
                      "what": "stream of independent C3-shaped matvecs, 3 in flight on 3 CUDA streams "
                              "(own workspaces), device-resident inputs; CUDA events on the calling stream"}
        del others[1:]
    elif args.plan == "coset":
        from paper_1402_5287_b200 import dist as hkdist
        cs = hkdist.CosetStream(kind, (a, sa, x, sx), P, slots=3,
                                p2p=(getattr(sh, "p2p", False) or "auto") if sh_verified_p2p else False,
                                sliced=sh.sliced)
        probs = [(a, sa, x, sx)] * n_tp
        cs.run(probs[:6])
        torch.cuda.synchronize()
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        cs.run(probs)
        c1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        tt = torch.tensor([c0.elapsed_time(c1)], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        cms = float(tt.item()) / n_tp
        throughput = {"value": 1000.0 / cms, "unit": UNIT, "ms_per_matvec": cms, "matvecs": n_tp,
                      "in_flight": 3, "p2p": cs.p2p, "sliced": cs.sliced,
                      "launches_per_rank": (4 if cs.sliced else 3) * n_tp,
                      "what": "CosetStream: stream of independent matvecs over the sigma-coset shards, 3 slots, "
                              "exchanges on a communication stream overlapping the next matvec's K1/K2; "
                              "CUDA events, max over ranks"}
        del cs

    # ---- F4 (secondary): the same matvec with y rounded back to the input format (L+1 limbs)
    rounded = None
    if rank == 0 and world == 1:
        L = plan["L"]
        yr = (torch.empty((n, L + 1), dtype=torch.int64, device=dev),
              torch.empty((n,), dtype=torch.int8, device=dev))
        wsr = hk.Workspace(kind, n, P)
        for _ in range(W):
            hk.matvec(kind, a, sa, x, sx, P, out=yr, ws=wsr, check=False, rounded=True)
        torch.cuda.synchronize()
        r0_ = torch.cuda.Event(enable_timing=True)
        r1_ = torch.cuda.Event(enable_timing=True)
        r0_.record(stream)
        for _ in range(K):
            hk.matvec(kind, a, sa, x, sx, P, out=yr, ws=wsr, check=False, rounded=True)
        r1_.record(stream)
        torch.cuda.synchronize()
        if wsr.status() != hk.HK_OK:
            raise SystemExit("bench: rounded-matvec status not OK")
        rms = r0_.elapsed_time(r1_) / K
        rounded = {"value": 1000.0 / rms, "unit": UNIT, "ms_per_step": rms,
                   "what": "hk_matvec_rounded: y = round_half_even(Y / 2^P), L+1 limbs (SURVEY 8(f) F4)"}
        del wsr, yr

    # ---- F3 (secondary): the same matvec through the exact FP64 double-FFT path (hk_fft_matvec;
    # the paper's decomposition approach, with Percival's bound)
    fp64 = None
    if rank == 0 and world == 1:
        fpl = hk.fft_plan(kind, n, P)
        fws = hk.FftWorkspace(kind, n, P)
        yf = (torch.empty((n, plan["Ly"]), dtype=torch.int64, device=dev),
              torch.empty((n,), dtype=torch.int8, device=dev))
        hk.fft_matvec(kind, a, sa, x, sx, P, out=yf, ws=fws)
        okf, whyf = verify_y(kind, am, asg, xm, xsg, yf[0], yf[1], 0, 1, None, dev)
        if not okf:
            raise SystemExit(f"bench: FP64-FFT y fails its fingerprints ({whyf})")
        Kf = max(3, min(K, 20))
        for _ in range(2):
            hk.fft_matvec(kind, a, sa, x, sx, P, out=yf, ws=fws, check=False)
        f0_, f1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0_.record(stream)
        for _ in range(Kf):
            hk.fft_matvec(kind, a, sa, x, sx, P, out=yf, ws=fws, check=False)
        f1_.record(stream)
        torch.cuda.synchronize()
        if fws.status() != hk.HK_OK:
            raise SystemExit("bench: FP64-FFT status not OK")
        fms = f0_.elapsed_time(f1_) / Kf
        N1f, N2f = 1 << fpl["log_n1"], 1 << fpl["log_n2"]
        bfl = ((fpl["a_count"] + 2 * n) * (N2f // 2) * fpl["log_n2"] +
               3 * N2f * (N1f // 2) * fpl["log_n1"])  # complex radix-2 butterflies
        dp_ops = 10 * bfl  # 4 DMUL + 2 DADD (complex product) + 4 DADD per butterfly, no FMA
        nsm_ = torch.cuda.get_device_properties(dev).multi_processor_count
        smx_ = float(json.load(open(PEAKS_FILE)).get("sm_max_mhz", 1965.0)) if os.path.exists(PEAKS_FILE) else 1965.0
        dp_peak = nsm_ * 56 * smx_ * 1e6  # FP64 lanes / clk / SM measured (profiles/r01/micro_fp64.log)
        fp64 = {"value": 1000.0 / fms, "unit": UNIT, "ms_per_step": fms, "steps": Kf,
                "plan": {k_: fpl[k_] for k_ in ("w", "Ls", "log_n1", "log_n2", "bound")},
                "verified": "fingerprints of every row (mod 3 primes) before timing",
                "fp64_ops": dp_ops, "fp64_peak_ops_s": dp_peak,
                "fp64_frac": dp_ops / (fms * 1e-3) / dp_peak,
                "what": "hk_fft_matvec: balanced w-bit digits, 2-D complex FP64 FFT convolution with a proven "
                        "< 1/2 error (Percival), rint, carry (SURVEY 8(f) F3); ops = 10 per complex butterfly "
                        "against 56 FP64 lanes/clk/SM"}
        del fws, yf

    # ---- e2e through the host-buffer C-ABI call (N = 1 workload per rank)
    e2e = None
    if rank == 0 and not args.no_e2e and world == 1:
        pa = torch.from_numpy(am.view(np.int64)).pin_memory()
        ps = torch.from_numpy(asg).pin_memory()
        px = torch.from_numpy(xm.view(np.int64)).pin_memory()
        pxs = torch.from_numpy(xsg).pin_memory()
        Ly = plan["Ly"]
        py = torch.empty((n, Ly), dtype=torch.int64).pin_memory()
        pys = torch.empty((n,), dtype=torch.int8).pin_memory()
        # (i) latency of one synchronous call (hk_matvec_host: chunked H2D/K1 and K3/D2H overlap)
        wsh = hk.Workspace(kind, n, P, flags=hk.WS_STAGING)
        for _ in range(2):
            hk.matvec_host(kind, pa, ps, px, pxs, P, out=(py, pys), ws=wsh)
        torch.cuda.synchronize()
        Kl = 5
        t0 = time.perf_counter()
        for _ in range(Kl):
            hk.matvec_host(kind, pa, ps, px, pxs, P, out=(py, pys), ws=wsh)
        ms_lat = (time.perf_counter() - t0) * 1e3 / Kl
        del wsh
        # (ii) throughput: a stream of calls through HostPipeline (hk_matvec_host_async, 3 lanes);
        # every step copies its own a, x in and its y (+ status) out inside the timed region
        depth = 3
        pipe = hk.HostPipeline(kind, n, P, depth=depth)
        outs = [(torch.empty((n, Ly), dtype=torch.int64).pin_memory(),
                 torch.empty((n,), dtype=torch.int8).pin_memory()) for _ in range(depth)]
        for i in range(2 * depth):
            pipe.submit(pa, ps, px, pxs, outs[i % depth])
        pipe.drain()
        Ke = max(3, min(K, 30))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(Ke):
            pipe.submit(pa, ps, px, pxs, outs[i % depth])
        pipe.drain()
        ms_e2e = (time.perf_counter() - t0) * 1e3 / Ke
        h2d = am.nbytes + asg.nbytes + xm.nbytes + xsg.nbytes
        d2h = n * Ly * 8 + n + 4
        e2e = {"value": 1000.0 / ms_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ms_e2e, "steps": Ke,
               "api": f"HostPipeline(depth={depth}).submit -> hk_matvec_host_async (pinned host "
                      "buffers; lanes overlap one call's copies with another's kernels)",
               "timing": "host wall clock from first submit to drain (all device work complete)",
               "latency_ms_single_call": ms_lat,
               "single_call_api": "hk_matvec_host (synchronous)",
               "pcie": pcie_roofline(h2d, d2h, ms_e2e, dev)}
        del pipe

    # ---- e2e at N > 1: every step each rank copies its (replicated) a and x from pinned host memory,
    # the sharded step runs, rank 0 reads y back; host wall clock between barriers, max over ranks
    if world > 1 and not args.no_e2e:
        pa = torch.from_numpy(am.view(np.int64)).pin_memory()
        ps = torch.from_numpy(asg).pin_memory()
        px = torch.from_numpy(xm.view(np.int64)).pin_memory()
        pxs = torch.from_numpy(xsg).pin_memory()
        ym_h, ys_h = None, None
        Ke = max(3, min(K, 20))

        def e2e_step():
            a.copy_(pa, non_blocking=True)
            sa.copy_(ps, non_blocking=True)
            x.copy_(px, non_blocking=True)
            sx.copy_(pxs, non_blocking=True)
            step()
            if rank == 0:
                y_dev, s_dev = sh.result()
                nonlocal ym_h, ys_h
                if ym_h is None:
                    ym_h = torch.empty(y_dev.shape, dtype=y_dev.dtype).pin_memory()
                    ys_h = torch.empty(s_dev.shape, dtype=s_dev.dtype).pin_memory()
                ym_h.copy_(y_dev, non_blocking=True)
                ys_h.copy_(s_dev, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(2):
            e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(Ke):
            e2e_step()
        dist.barrier()
        tt = torch.tensor([(time.perf_counter() - t0) * 1e3 / Ke], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_e2e = float(tt.item())
        Ly = plan["Ly"]
        e2e = {"value": 1000.0 / ms_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(world * (am.nbytes + asg.nbytes + xm.nbytes + xsg.nbytes)),
               "d2h_bytes_per_step": int(n * Ly * 8 + n), "ms_per_step": ms_e2e, "steps": Ke,
               "api": "every rank: H2D of a, x into its device inputs; the sharded step; rank 0: D2H of y",
               "timing": "host wall clock between barriers, max over ranks (synchronous steps)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline: integer issue slots, 128 thread-instr / clk / SM
    cnt = alg_counts(plan)
    sm_cnt = survey_model(plan)
    peaks = {}
    if os.path.exists(PEAKS_FILE):
        peaks = json.load(open(PEAKS_FILE))
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_bfly = nsm * BFLY_PER_CLK_SM * sm_max * 1e6 / 1e12
    peak_tinstr = nsm * LANES_PER_SM * sm_max * 1e6 / 1e12
    hbm_peak = float(peaks.get("hbm_gbs", 6549.4))
    io_bytes, all_bytes = alg_bytes(plan)
    t_alu = sm_cnt["total"] / (peak_tinstr * 1e12)
    t_hbm = all_bytes / (hbm_peak * 1e9)
    t_roof = max(t_alu, t_hbm)
    k2_ms = stage_ms[1]
    traffic = None
    tf = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(wl["name"])
        except (ValueError, OSError):
            traffic = None
    single = world == 1
    achieved = sm_cnt["K2"] / (k2_ms * 1e-3) / 1e12 if single else None
    roof = {"bound": "alu", "kernel": "k2_column", "achieved": achieved, "peak": peak_tinstr,
            "unit": "T thread-instr/s", "frac": (achieved / peak_tinstr) if achieved else None,
            "traffic": traffic,
            "peak_source": f"derived (SURVEY.md 8(d)): {nsm} SMs x {LANES_PER_SM} thread-instr/clk/SM "
                           f"(4 SMSPs x 32 lanes issue limit) x {sm_max:.0f} MHz (MEASURED_PEAKS.json "
                           "sm_max_mhz)",
            "algorithmic_per_launch": sm_cnt["K2"],
            "per_unit": (f"SURVEY.md 8(d): {S_BFLY} per butterfly, {S_PW} per pointwise product "
                         "(K2: 3 column NTTs of N1 points per (prime, sigma) column, 5 N2 columns, full "
                         "transforms, no pruning credit)"),
            "kernel_ms": k2_ms, "kernel_share_of_step": k2_ms / ms_step,
            "step_frac": (t_roof / (ms_step * 1e-3)) if single else (t_roof / world) / (ms_step * 1e-3),
            "step": {"T_roof_us": t_roof * 1e6, "T_alu_us": t_alu * 1e6, "T_hbm_us": t_hbm * 1e6,
                     "I_alg": sm_cnt["total"], "B_alg": all_bytes, "T_measured_us": ms_step * 1e3,
                     "definition": "SURVEY.md 8(d): T_roof = max(I_alg / (128 N_SM f), B_alg / HBM peak); "
                                   "step_frac = T_roof / T_measured (at N > 1: T_roof / N)",
                     "constants": {"butterfly": S_BFLY, "pointwise": S_PW, "slice_residue": S_RES,
                                   "crt": C_CRT, "carry_limb": C_CARRY,
                                   "survey_estimates": {"crt": S_CRT_SURVEY, "carry_limb": S_CARRY_SURVEY}},
                     "counts": {k_: sm_cnt[k_] for k_ in ("butterflies", "pointwise", "residues", "crt",
                                                          "carry_limbs")}}}
    if single:  # the same model per kernel (CUDA-event stage times)
        roof["kernels"] = {name: {"I_alg": sm_cnt[key], "kernel_ms": ms_,
                                  "frac": sm_cnt[key] / (peak_tinstr * 1e12) / (ms_ * 1e-3)}
                           for name, key, ms_ in (("k1_slice_rowntt", "K1", stage_ms[0]),
                                                  ("k2_column", "K2", stage_ms[1]),
                                                  ("k3_finish", "K3", stage_ms[2]))}
        roof["kernels"]["k3_finish"]["frac_survey_constants"] = (
            sm_cnt["K3_survey_constants"] / (peak_tinstr * 1e12) / (stage_ms[2] * 1e-3))
        t_alu_s = (sm_cnt["total"] - sm_cnt["K3"] + sm_cnt["K3_survey_constants"]) / (peak_tinstr * 1e12)
        roof["step"]["step_frac_survey_constants"] = max(t_alu_s, t_hbm) / (ms_step * 1e-3)
        ach_bfly = cnt["k2_bfly_eq"] / (k2_ms * 1e-3) / 1e12
        roof["pipe_model"] = {
            "what": "secondary: K2 in GS-butterfly equivalents against the FMA-pipe limit (IMAD.HI 4 clk, "
                    "IMAD 2 clk per warp per SMSP: GS 8, CT 9, Montgomery 10 pipe clocks)",
            "achieved": ach_bfly, "peak": peak_bfly, "unit": "T GS-butterfly-eq/s", "frac": ach_bfly / peak_bfly,
            "vs_microbenchmark": (cnt["bf_col_fwd"] / MICRO_GS + cnt["bf_col_inv"] / MICRO_CT +
                                  cnt["pointwise"] * C_MONT / C_GS / MICRO_GS) / (nsm * sm_max * 1e6) /
                                 (k2_ms * 1e-3),
            "vs_microbenchmark_note": "K2 time vs its butterflies at the register-resident loop rates of "
                                      "scripts/micro_bfly.cu (GS 12.07, CT 11.22 per clk per SM)"}
    roof["hbm_check"] = {"alg_bytes_per_step": all_bytes,
                         "achieved_gbs": all_bytes / (ms_step * 1e-3) / 1e9, "peak_gbs": hbm_peak}

    cb = None
    if not args.no_cpu:
        cb = cpu_baseline(wl, y_gpu=hk.to_host(prob.y_mag, prob.y_sign) if world == 1 else None)
        if world == 1 and cb["gpu_rows_differing"]:
            raise SystemExit(f"bench: {cb['gpu_rows_differing']} sampled rows differ from the oracle")

    value = 1000.0 / ms_step  # one matvec per step for the whole job
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded SplitMix64 mantissas, BASELINE configs recipe)",
        "config": workload_config(wl),
        "plan": {k: plan[k] for k in ("w", "Ls", "log_n1", "log_n2", "k_primes", "margin_bits")},
        "parallelism": "single GPU" if world == 1 else (
            (f"sigma-coset x{world}" + (" sliced (each rank slices 1/G of the positions, slice "
                                         "all-to-all before K2)" if getattr(sh, "sliced", False) else "")
             + ": " + ("exchanges fused into K1/K2/K3 stores over peer memory "
                                          "(symmetric memory, NVLink) + device barriers"
                                          if getattr(sh, "p2p", False) else
                                          "NCCL all-to-all + all-gather"))
            if args.plan == "coset" else f"row-block x{world} + NCCL all-gather"),
        "launch": ("host call per step" if (world > 1 or args.no_graph) else
                   "CUDA graph replay per step (Problem.capture: the same K1/K2/K3 launches)"),
        "stages_ms": dict(zip(stage_names, stage_ms)),
        "roofline": roof,
        "verification": verification,
        "cpu_baseline": cb,
        "e2e": e2e,
        "warm_a": warm,
        "rounded": rounded,
        "fp64_fft": fp64,
        "throughput": throughput,
        "gpu_launches": launches_per_step * K,
        "clocks": clocks,
        "library": hk.library_path(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
