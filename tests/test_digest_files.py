"""The committed oracle digests (tests/golden/digests/, written by scripts/oracle_digests.py from
``oracle/`` alone) are well-formed and belong to today's seeded inputs: one 64-bit digest per output
row of every BASELINE config, none missing, the row file pinned by its SHA-256 where the json
carries one, and the input SHA-256 equal to the generator's (PAPER.md P:50-90 defines the product
whose rows they digest; the GPU comparison is tests/test_gpu_digests.py)."""
import hashlib
import json
import os
import re

import numpy as np
import pytest

import hkinputs as gen

DIG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "digests")
NAMES = ("C1", "C2", "C3", "C4", "C5T", "C5C")


@pytest.mark.parametrize("name", NAMES)
def test_digest_file_is_complete(name):
    meta = json.load(open(os.path.join(DIG, f"{name}.json")))
    c = gen.CONFIGS[name]
    assert (meta["kind"], meta["n"], meta["P"], meta["seed"]) == (c["kind"], c["n"], c["P"], c["seed"])
    text = open(os.path.join(DIG, f"{name}.rows")).read()
    rows = text.split()
    assert len(rows) == meta["rows"] == c["n"]  # square problems: one output row per entry of x
    assert all(re.fullmatch(r"[0-9a-f]{16}", r) for r in rows), "a row without an oracle digest"
    assert meta.get("rows_missing", 0) == 0
    if meta.get("rows_sha256"):
        assert hashlib.sha256(text.encode()).hexdigest() == meta["rows_sha256"]
    assert meta.get("y_sha256") or meta.get("rows_sha256")


@pytest.mark.parametrize("name", NAMES)
def test_digest_inputs_are_todays(name):
    meta = json.load(open(os.path.join(DIG, f"{name}.json")))
    h = hashlib.sha256()
    for v in gen.config_inputs(name):
        h.update(np.ascontiguousarray(v).tobytes())
    assert h.hexdigest() == meta["input_sha256"], "the seeded generator changed since the oracle run"
