"""Full-size oracle digests for the BASELINE configs (test infrastructure; calls only ``oracle/``
and ``hkinputs/``, never the CUDA path).

For each config it regenerates the seeded inputs, runs the C oracle over EVERY output row (in
row chunks, checkpointed under ``.oracle_cache/`` so an interrupted run resumes), and writes

  tests/golden/digests/<config>.json   -- config, seed, recipe, input SHA-256, SHA-256 of the
                                          whole y (y_mag bytes then y_sign bytes), row count
  tests/golden/digests/<config>.rows   -- one line per output row: the first 16 hex digits of
                                          SHA-256(y_mag[i] bytes || y_sign[i] byte)

so that ``tests/test_gpu_digests.py`` can compare the GPU's y with the oracle's byte for byte
(via the digest) and name the first differing rows, without re-running hours of oracle work.
The oracle computes the plain definition; nothing here comes
from the CUDA path.

  python scripts/oracle_digests.py C2 C5T C5C C3 C4 --threads 7
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hkinputs as gen  # noqa: E402
import oracle  # noqa: E402

CACHE = os.path.join(ROOT, ".oracle_cache")
OUT = os.path.join(ROOT, "tests", "golden", "digests")


def input_sha256(am, asg, xm, xsg) -> str:
    h = hashlib.sha256()
    for v in (am, asg, xm, xsg):
        h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()


def row_digest(ym_row: np.ndarray, ys_val: np.int8) -> str:
    return hashlib.sha256(ym_row.tobytes() + np.int8(ys_val).tobytes()).hexdigest()[:16]


def run(name: str, threads: int, chunk: int) -> None:
    c = gen.CONFIGS[name]
    kind, n, P = c["kind"], c["n"], c["P"]
    am, asg, xm, xsg = gen.config_inputs(name)
    isha = input_sha256(am, asg, xm, xsg)
    cdir = os.path.join(CACHE, f"{name}_{isha[:16]}")
    os.makedirs(cdir, exist_ok=True)
    t0 = time.time()
    for r0 in range(0, n, chunk):
        f = os.path.join(cdir, f"rows_{r0:06d}.npz")
        if os.path.exists(f):
            continue
        rows = np.arange(r0, min(n, r0 + chunk), dtype=np.int64)
        t1 = time.time()
        ym, ys = oracle.matvec(kind, P, am, asg, xm, xsg, rows=rows, threads=threads)
        np.savez(f + ".tmp.npz", y_mag=ym, y_sign=ys)
        os.replace(f + ".tmp.npz", f)
        print(f"{name}: rows {r0}..{rows[-1]} in {time.time() - t1:.1f} s", flush=True)
    # assemble in row order
    h = hashlib.sha256()
    mags, signs, lines = [], [], []
    for r0 in range(0, n, chunk):
        d = np.load(os.path.join(cdir, f"rows_{r0:06d}.npz"))
        ym, ys = d["y_mag"], d["y_sign"]
        mags.append(ym)
        signs.append(ys)
        lines.extend(row_digest(ym[i], ys[i]) for i in range(ym.shape[0]))
    y_mag = np.concatenate(mags)
    y_sign = np.concatenate(signs)
    assert y_mag.shape == (n, gen.n_out_limbs(P)) and y_sign.shape == (n,)
    h.update(y_mag.tobytes())
    h.update(y_sign.tobytes())
    os.makedirs(OUT, exist_ok=True)
    meta = dict(config=name, kind=kind, n=n, P=P, seed=c["seed"], recipe=c["recipe"],
                generator="hkinputs SplitMix64 counter generator (SURVEY §8(d))",
                input_sha256=isha, y_sha256=h.hexdigest(), rows=n,
                row_digest="first 16 hex of SHA-256(y_mag[i] || y_sign[i])",
                produced_by="scripts/oracle_digests.py (oracle/hk_oracle.c, all rows)",
                oracle_threads=threads)
    with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
        fh.write("\n")
    with open(os.path.join(OUT, f"{name}.rows"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print(f"{name}: done, y sha256 {h.hexdigest()} ({time.time() - t0:.0f} s this run)", flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--chunk", type=int, default=0, help="rows per checkpoint (default by size)")
    args = ap.parse_args()
    for name in args.configs:
        n = gen.CONFIGS[name]["n"]
        run(name, args.threads, args.chunk or (128 if n > 4096 else 512))


if __name__ == "__main__":
    main()
