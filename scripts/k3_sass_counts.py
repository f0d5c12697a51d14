"""SASS instruction counts of K3 (k3_finish) per CRT coefficient and per carry limb -- the c_CRT and
c_carry constants of the SURVEY.md 8(d) roofline (which the survey left as estimates, 110 and 25,
"the builder recounts them from its own SASS once").

    python scripts/k3_sass_counts.py [--logn2 10 --ch 13] [--cubin path]

Compiles paper_1402_5287_b200/csrc/hk_ntt.cu to a cubin (unless --cubin is given), extracts
k3_finish<LOGN2, CH> and splits it at its CTA barriers (BAR.SYNC / BAR.RED):
  phase 2 -> 3 (after the inverse slice NTT): the Garner loop, one coefficient per iteration:
           c_CRT = instructions of that loop body;
  phase 3 -> the barrier before the y staging store: the carry phase (gather, local carries,
           lookahead scan, final limbs, sign), straight-line code over the CH limbs of a thread:
           c_carry = its instructions / CH (the per-warp sequential tail over the R rows is included).
Static counts of the code each thread executes once per coefficient / limb.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_of(cubin: str, func: str) -> list[tuple[int, str]]:
    out = subprocess.check_output(["cuobjdump", "-sass", "-fun", func, cubin], text=True)
    ins = []
    for ln in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(3)))
    return ins


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn2", type=int, default=10)
    ap.add_argument("--ch", type=int, default=13)
    ap.add_argument("--cubin", default=None)
    args = ap.parse_args()
    cubin = args.cubin
    if cubin is None:
        os.makedirs(os.path.join(ROOT, ".oracle_cache", "sass"), exist_ok=True)
        cubin = os.path.join(ROOT, ".oracle_cache", "sass", "hk_ntt.cubin")
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-cubin",
                               "-o", cubin, os.path.join(ROOT, "paper_1402_5287_b200", "csrc", "hk_ntt.cu")])
    func = f"_ZN2hk9k3_finishILi{args.logn2}ELi{args.ch}EEEvNS_6ParamsE"
    ins = sass_of(cubin, func)
    bars = [i for i, (_, op) in enumerate(ins) if op.startswith("BAR.SYNC") or op.startswith("BAR.RED")]
    # barrier order: load, DIT pass 1, DIT pass 2, Garner, carry (local -> s_ecarry), scan (warp
    # totals), scan (warp carries), final limbs (-> ybuf), ybuf staged, ...
    garner = ins[bars[2] + 1:bars[3]]
    addrs = [a for a, _ in garner]
    best = None  # the Garner loop: the largest backward-branch range inside the phase
    text = subprocess.check_output(["cuobjdump", "-sass", "-fun", func, cubin], text=True)
    for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+(?:@!?U?P\w+\s+)?BRA\s+`?\(?\.?L?_?x?_?\w*\)?`?\s*0x([0-9a-f]+)", text):
        src, dst = int(m.group(1), 16), int(m.group(2), 16)
        if dst < src and addrs and addrs[0] <= dst and src <= addrs[-1]:
            n = sum(1 for a in addrs if dst <= a <= src)
            if best is None or n > best[0]:
                best = (n, dst, src)
    c_crt = best[0] if best else None
    # carry phase: from the Garner barrier to the barrier after which the y rows are staged (the
    # 4th barrier after it: local carries | warp totals | warp carries | final limbs)
    carry = ins[bars[3] + 1:bars[7]]
    c_carry = len(carry) / args.ch
    res = {"kernel": f"k3_finish<{args.logn2},{args.ch}>", "c_crt_instr_per_coefficient": c_crt,
           "garner_loop": None if best is None else [hex(best[1]), hex(best[2])],
           "carry_phase_instr": len(carry), "limbs_per_thread": args.ch,
           "c_carry_instr_per_limb": round(c_carry, 1), "barriers": len(bars)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    sys.exit(main())
