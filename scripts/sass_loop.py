"""Opcode histogram of the innermost loops of a kernel's SASS (cuobjdump -sass output on stdin):
every backward branch target..branch range, largest first.  Dev tool for instruction-mix checks."""
import re
import sys
from collections import Counter

lines = sys.stdin.read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\d+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
loops = []
for i, (addr, op, rest) in enumerate(ins):
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", rest)
        if t and int(t.group(1), 16) < addr:
            tgt = int(t.group(1), 16)
            body = [o for (a, o, _) in ins if tgt <= a <= addr]
            loops.append((len(body), tgt, addr, Counter(body)))
loops.sort(reverse=True)
for n, tgt, addr, c in loops[: int(sys.argv[1]) if len(sys.argv) > 1 else 1]:
    print(f"loop 0x{tgt:x}..0x{addr:x}: {n} instructions")
    for op, k in c.most_common(14):
        print(f"  {k:5d} {op}")
