#!/usr/bin/env python
"""Per-opcode executed-instruction and stall-sample breakdown of one kernel in an ncu report."""
import collections, csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if 'Source' in r and 'Instructions Executed' in r][0]
hdr = rows[hi]; si = hdr.index('Source'); ei = hdr.index('Instructions Executed')
wi = hdr.index('Warp Stall Sampling (All Samples)')
cnt = collections.Counter(); st = collections.Counter(); tot = 0; stot = 0
for r in rows[hi + 1:]:
    if len(r) <= max(ei, wi): continue
    try: n = int(r[ei]); w = int(r[wi])
    except ValueError: continue
    toks = r[si].strip().split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    cnt[op] += n; tot += n; st[op] += w; stot += w
print(f"{kre}: warp-inst {tot}, stall samples {stot}")
for k, v in cnt.most_common(18):
    print(f"  {k:26s} inst {v / tot * 100:5.1f}%  stall {st[k] / max(stot, 1) * 100:5.1f}%")
