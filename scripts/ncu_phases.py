#!/usr/bin/env python
"""Stall-sample / instruction shares of one kernel by source-line ranges of a file.
usage: ncu_phases.py REP KERNEL_RE FILE name:lo-hi [name:lo-hi ...]   (other files -> their name)"""
import csv, io, os, subprocess, sys
rep, kre, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[4:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
tot, hdr, cur = {}, None, ""
for r in csv.reader(io.StringIO(raw)):
    if not r: continue
    if r[0] == "File Path": cur = os.path.basename(r[1]); continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0]: continue
    try:
        w = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = int(r[hdr.index("Instructions Executed")] or 0); ln = int(r[0])
    except (ValueError, IndexError):
        continue
    ph = cur
    if cur == fname:
        ph = next((nm for nm, lo, hi in ranges if lo <= ln <= hi), f"{cur}:other")
    a = tot.setdefault(ph, [0, 0]); a[0] += w; a[1] += n
W = sum(v[0] for v in tot.values()) or 1; N = sum(v[1] for v in tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} stall {v[0] / W * 100:5.1f}%  inst {v[1] / N * 100:5.1f}%")
