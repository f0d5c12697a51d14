#!/usr/bin/env python
"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples and executed
instructions (needs -lineinfo builds and --import-source on).  usage: ncu_lines.py REP KERNEL_RE [N]"""
import csv, io, os, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
recs, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(raw)):
    if not r: continue
    if r[0] == "File Path": fname = os.path.basename(r[1]); continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0]: continue
    try:
        w = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    recs.append((w, n, f"{fname}:{r[0]}", r[1].strip()[:100]))
tw = sum(x[0] for x in recs) or 1; tn = sum(x[1] for x in recs) or 1
print(f"{kre}: stall samples {tw}, warp-inst {tn}")
for w, n, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{w / tw * 100:5.1f}% stall {n / tn * 100:5.1f}% inst  {ln}: {src}")
