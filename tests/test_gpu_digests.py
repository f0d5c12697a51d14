"""Full-size bit-exact parity on every BASELINE config (north_star: "bit-exact agreement with the
oracle on all five configs"; PAPER.md P:50-90 defines the product).

The oracle's y over EVERY row of C2, C3, C4, C5-Toeplitz and C5-circulant takes 1.5 min to 28 core-hours
of host time, so ``scripts/oracle_digests.py`` (which calls only ``oracle/`` and ``hkinputs/``)
ran it once and committed, per config, the SHA-256 of the whole y and a 64-bit digest of every
row under ``tests/golden/digests/``.  Here the GPU computes y in the launch configuration
bench.py times (``Problem.run``, all three kernels) and must reproduce the whole-y digest
byte for byte; on a mismatch the per-row digests name the first differing rows.  The input
SHA-256 pins the seeded generator, so a changed generator cannot silently pass."""
import hashlib
import json
import os

import numpy as np
import pytest

import hkinputs as gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DIG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "digests")
CONFIGS = [c for c in ("C1", "C2", "C3", "C4", "C5T", "C5C")
           if os.path.exists(os.path.join(DIG, f"{c}.json"))]


def input_sha256(am, asg, xm, xsg) -> str:
    h = hashlib.sha256()
    for v in (am, asg, xm, xsg):
        h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()


def row_digests(ym, ys):
    return [hashlib.sha256(ym[i].tobytes() + ys[i:i + 1].tobytes()).hexdigest()[:16]
            for i in range(ym.shape[0])]


def _check(name, meta, ym, ys):
    """Whole-y SHA-256 when the oracle run kept every limb; otherwise (C4, split between hosts,
    scripts/oracle_digests.py --dig-dir) every row's 64-bit digest, pinned by rows_sha256."""
    want_rows = open(os.path.join(DIG, f"{name.split()[0]}.rows")).read()
    if meta.get("rows_sha256"):
        assert hashlib.sha256(want_rows.encode()).hexdigest() == meta["rows_sha256"]
    want = want_rows.split()
    assert len(want) == ym.shape[0] == meta["rows"]
    if meta.get("y_sha256"):
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(ym).tobytes())
        h.update(np.ascontiguousarray(ys).tobytes())
        if h.hexdigest() == meta["y_sha256"]:
            return
    got = row_digests(ym, ys)
    missing = [i for i, w in enumerate(want) if w == "-" * 16]  # an unfinished oracle run (--partial)
    assert len(missing) == meta.get("rows_missing", 0)
    bad = [i for i, (g, w) in enumerate(zip(got, want)) if g != w and w != "-" * 16]
    if bad or not meta.get("y_sha256"):
        assert not bad, f"{name}: y differs from the oracle's in {len(bad)} rows, first {bad[:8]}"
        return
    pytest.fail(f"{name}: every row digest matches but the whole-y SHA-256 does not")


@pytest.fixture(scope="module")
def hk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1402_5287_b200 as hk
    return hk


@pytest.mark.parametrize("name", CONFIGS)
def test_config_matches_oracle_digest(hk, name):
    meta = json.load(open(os.path.join(DIG, f"{name}.json")))
    c = gen.CONFIGS[name]
    kind, n, P = c["kind"], c["n"], c["P"]
    am, asg, xm, xsg = gen.config_inputs(name)
    assert input_sha256(am, asg, xm, xsg) == meta["input_sha256"], "generator changed"
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    prob = hk.Problem(kind, a, sa, x, sx, P)  # bench.py's launch configuration (K1, K2, K3)
    prob.run()
    torch.cuda.synchronize()
    assert prob.status() == hk.HK_OK
    ym, ys = hk.to_host(*prob.result())
    _check(name, meta, ym, ys)
    # the bench's timed steps: the same step replayed from a CUDA graph (Problem.capture)
    prob.y_mag.fill_(-1)
    prob.y_sign.fill_(7)
    prob.capture()
    prob.replay()
    torch.cuda.synchronize()
    assert prob.status() == hk.HK_OK
    ym, ys = hk.to_host(*prob.result())
    _check(name + " (graph replay)", meta, ym, ys)
