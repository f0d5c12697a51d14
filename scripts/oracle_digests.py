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

C4 (n = 16384: about 27 core-hours) is split between hosts: ``--chunks A:B`` computes only chunk
indices A..B-1 (``--reverse`` walks them from the top) and ``--dig-dir D`` writes each chunk's row
digests as ``D/rows_XXXXXX.dig`` (16 hex per line, 2 KB per chunk instead of 1 MB of limbs), so a
remote host can ship its share back; ``--assemble --dig-dir D ...`` then writes the config's
digest files from every chunk's .npz or .dig.  When some chunks exist only as digests the whole-y
SHA-256 cannot be formed: the json then carries ``y_sha256: null`` and ``rows_sha256`` (SHA-256 of
the .rows file), and tests/test_gpu_digests.py compares every row's digest instead.  ``--partial``
assembles an unfinished run: rows nobody computed carry a placeholder, ``rows_missing`` counts them.
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


MISSING = "-" * 16  # placeholder digest of a row no host has computed yet (--partial)


def run(name: str, threads: int, chunk: int, chunks=None, reverse=False, dig_dir=None,
        assemble=True, partial=False) -> None:
    c = gen.CONFIGS[name]
    kind, n, P = c["kind"], c["n"], c["P"]
    am, asg, xm, xsg = gen.config_inputs(name)
    isha = input_sha256(am, asg, xm, xsg)
    cdir = os.path.join(CACHE, f"{name}_{isha[:16]}")
    os.makedirs(cdir, exist_ok=True)
    if dig_dir:
        os.makedirs(dig_dir, exist_ok=True)
    t0 = time.time()
    starts = list(range(0, n, chunk))
    todo = starts if chunks is None else starts[chunks[0]:chunks[1]]
    for r0 in (reversed(todo) if reverse else todo):
        f = os.path.join(cdir, f"rows_{r0:06d}.npz")
        fd = os.path.join(dig_dir, f"rows_{r0:06d}.dig") if dig_dir else None
        if os.path.exists(f) or (fd and os.path.exists(fd)):
            continue
        rows = np.arange(r0, min(n, r0 + chunk), dtype=np.int64)
        t1 = time.time()
        ym, ys = oracle.matvec(kind, P, am, asg, xm, xsg, rows=rows, threads=threads)
        if fd:
            with open(fd + ".tmp", "w") as fh:
                fh.write("\n".join(row_digest(ym[i], ys[i]) for i in range(len(rows))) + "\n")
            os.replace(fd + ".tmp", fd)
        else:
            np.savez(f + ".tmp.npz", y_mag=ym, y_sign=ys)
            os.replace(f + ".tmp.npz", f)
        print(f"{name}: rows {r0}..{rows[-1]} in {time.time() - t1:.1f} s", flush=True)
    if not assemble:
        return
    # assemble in row order, from the limbs where this host has them, else from shipped digests
    h = hashlib.sha256()
    mags, signs, lines = [], [], []
    whole = True
    for r0 in starts:
        f = os.path.join(cdir, f"rows_{r0:06d}.npz")
        if os.path.exists(f):
            d = np.load(f)
            ym, ys = d["y_mag"], d["y_sign"]
            assert ym.shape == (min(n, r0 + chunk) - r0, gen.n_out_limbs(P))
            mags.append(ym)
            signs.append(ys)
            lines.extend(row_digest(ym[i], ys[i]) for i in range(ym.shape[0]))
        else:
            fd = os.path.join(dig_dir, f"rows_{r0:06d}.dig") if dig_dir else None
            if fd and os.path.exists(fd):
                got = open(fd).read().split()
            elif partial:  # an unfinished run: the test checks the rows that exist
                got = [MISSING] * (min(n, r0 + chunk) - r0)
            else:
                raise FileNotFoundError(f"chunk {r0}: neither limbs nor digests (use --partial)")
            assert len(got) == min(n, r0 + chunk) - r0, f"chunk {r0}: {len(got)} digests"
            lines.extend(got)
            whole = False
    assert len(lines) == n
    missing = sum(1 for d in lines if d == MISSING)
    if whole:
        y_mag = np.concatenate(mags)
        y_sign = np.concatenate(signs)
        assert y_mag.shape == (n, gen.n_out_limbs(P)) and y_sign.shape == (n,)
        h.update(y_mag.tobytes())
        h.update(y_sign.tobytes())
    rows_text = "\n".join(lines) + "\n"
    os.makedirs(OUT, exist_ok=True)
    meta = dict(config=name, kind=kind, n=n, P=P, seed=c["seed"], recipe=c["recipe"],
                generator="hkinputs SplitMix64 counter generator (SURVEY §8(d))",
                input_sha256=isha, y_sha256=h.hexdigest() if whole else None, rows=n,
                rows_missing=missing,
                rows_sha256=hashlib.sha256(rows_text.encode()).hexdigest(),
                row_digest="first 16 hex of SHA-256(y_mag[i] || y_sign[i])",
                produced_by="scripts/oracle_digests.py (oracle/hk_oracle.c, all rows)" +
                ("" if whole else "; row chunks computed on several hosts (--chunks/--dig-dir), "
                 "row digests only"),
                oracle_threads=threads)
    with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
        fh.write("\n")
    with open(os.path.join(OUT, f"{name}.rows"), "w") as fh:
        fh.write(rows_text)
    print(f"{name}: done, y sha256 {meta['y_sha256']} rows sha256 {meta['rows_sha256']} "
          f"({time.time() - t0:.0f} s this run)", flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--chunk", type=int, default=0, help="rows per checkpoint (default by size)")
    ap.add_argument("--chunks", default=None, help="A:B = compute only chunk indices A..B-1")
    ap.add_argument("--reverse", action="store_true", help="walk the chunks from the top")
    ap.add_argument("--dig-dir", default=None, help="write/read per-chunk row digests here")
    ap.add_argument("--no-assemble", action="store_true")
    ap.add_argument("--assemble", action="store_true", help="only assemble (compute nothing)")
    ap.add_argument("--partial", action="store_true",
                    help="assemble even if chunks are missing (their rows get a placeholder digest)")
    args = ap.parse_args()
    for name in args.configs:
        n = gen.CONFIGS[name]["n"]
        chunks = None
        if args.chunks:
            a, b = args.chunks.split(":")
            chunks = (int(a or 0), int(b) if b else None)
        if args.assemble:
            chunks = (0, 0)
        run(name, args.threads, args.chunk or (128 if n > 4096 else 512), chunks=chunks,
            reverse=args.reverse, dig_dir=args.dig_dir, assemble=not args.no_assemble,
            partial=args.partial)


if __name__ == "__main__":
    main()
