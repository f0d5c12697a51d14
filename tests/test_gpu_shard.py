"""GPU parity of the sigma-coset sharded path (SURVEY.md 8(e) plan P-2) through the C ABI
(hk_hankel_shard_forward / hk_hankel_shard_finish), bit-exact against the oracle.

There is one GPU here, so the G ranks run one after another in this process and the all-to-all
and all-gather are emulated by copies between their buffers (the same layouts NCCL moves in
paper_1402_5287_b200.dist.CosetShardedMatvec).  No rank waits on another inside a kernel."""
import numpy as np
import pytest

import hkinputs as gen
import oracle
from tests import fingerprint as fp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1402_5287_b200 as hk
    return hk


def sharded(hk, kind, G, am, asg, xm, xsg, P):
    n = xm.shape[0]
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    wss = [hk.ShardWorkspace(kind, n, P, G) for _ in range(G)]
    info = wss[0].info
    chunk, rpr, yr = info["chunk_words"], info["rows_per_rank"], info["y_rows"]
    Ly = hk.out_limbs(P)
    send = [torch.full((info["buffer_words"],), -1, dtype=torch.int32, device="cuda") for _ in range(G)]
    for g in range(G):
        hk.shard_forward(wss[g], g, a, sa, x, sx, send[g])
    # all-to-all: recv[r] chunk g = send[g] chunk r
    recv = [torch.cat([send[g][r * chunk:(r + 1) * chunk] for g in range(G)]) for r in range(G)]
    y_pads = []
    for g in range(G):
        ym = torch.full((yr, Ly), -7, dtype=torch.int64, device="cuda")
        ys = torch.full((yr,), 9, dtype=torch.int8, device="cuda")
        hk.shard_finish(wss[g], g, recv[g], ym, ys)
        y_pads.append((ym, ys))
    for g in range(G):
        assert wss[g].status() == hk.HK_OK
    # all-gather: block g of the padded y comes from rank g
    ym = torch.cat([y_pads[g][0][g * rpr:(g + 1) * rpr] for g in range(G)])
    ys = torch.cat([y_pads[g][1][g * rpr:(g + 1) * rpr] for g in range(G)])
    torch.cuda.synchronize()
    if kind == gen.TOEPLITZ:
        ym, ys = ym[yr - n:], ys[yr - n:]
    else:
        ym, ys = ym[:n], ys[:n]
    return hk.to_host(ym, ys)


@pytest.mark.parametrize("kind,n,P,G", [
    (0, 100, 4200, 2), (0, 100, 4200, 4), (0, 100, 4200, 8), (1, 77, 4200, 2), (1, 130, 8000, 8),
    (2, 64, 4200, 4), (2, 77, 9000, 8), (0, 1, 4200, 2), (0, 5, 17000, 8), (1, 3, 2500, 2),
    (0, 257, 2100, 2), (2, 128, 2100, 4)])
def test_coset_shards_match_oracle(hk, kind, n, P, G):
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=40 + n + G)
    got = sharded(hk, kind, G, am, asg, xm, xsg, P)
    want = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_coset_shards_carry_stress(hk):
    kind, n, P, G = 1, 96, 16608, 4
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=4, recipe="carry_stress")
    got = sharded(hk, kind, G, am, asg, xm, xsg, P)
    want = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("G", [2, 8])
def test_coset_shards_c2_fingerprints(hk, G):
    """BASELINE C2 (n = 1024, P = 33,216) over G shards: modular fingerprints of every row plus
    the oracle on sampled rows."""
    c = gen.CONFIGS["C2"]
    am, asg, xm, xsg = gen.config_inputs("C2")
    ym, ys = sharded(hk, c["kind"], G, am, asg, xm, xsg, c["P"])
    fp.check(c["kind"], am, asg, xm, xsg, ym, ys)
    rows = np.arange(0, c["n"], 97)
    wm, ws = oracle.matvec(c["kind"], c["P"], am, asg, xm, xsg, rows=rows)
    assert np.array_equal(ym[rows], wm) and np.array_equal(ys[rows], ws)


def test_shard_plan_rejects_bad_G(hk):
    for G in (3, 16, 0):
        with pytest.raises(hk.HKError):
            hk.shard_plan(0, 100, 4200, G)
    with pytest.raises(hk.HKError):  # N2 / G < 32 (P = 1000 -> N2 = 32)
        hk.shard_plan(0, 100, 1000, 2)


def sharded_p2p(hk, kind, G, am, asg, xm, xsg, P):
    """The peer-memory variant with G emulated ranks on one GPU: every rank's K2 writes straight
    into the other ranks' receive buffers and every rank's K3 into all ranks' y buffers (the
    pointers a multi-GPU run maps over NVLink are plain local pointers here)."""
    n = xm.shape[0]
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    wss = [hk.ShardWorkspace(kind, n, P, G) for _ in range(G)]
    info = wss[0].info
    yr, Ly = info["y_rows"], hk.out_limbs(P)
    recv = [torch.full((info["buffer_words"],), -1, dtype=torch.int32, device="cuda") for _ in range(G)]
    ym = [torch.full((yr, Ly), -7, dtype=torch.int64, device="cuda") for _ in range(G)]
    ys = [torch.full((yr,), 9, dtype=torch.int8, device="cuda") for _ in range(G)]
    rp = [t.data_ptr() for t in recv]
    for g in range(G):
        hk.shard_forward_p2p(wss[g], g, a, sa, x, sx, rp)
    torch.cuda.synchronize()  # the barrier between the phases
    for g in range(G):
        hk.shard_finish_p2p(wss[g], g, recv[g], [t.data_ptr() for t in ym], [t.data_ptr() for t in ys])
    torch.cuda.synchronize()
    for g in range(G):
        assert wss[g].status() == hk.HK_OK
    outs = []
    for d in range(G):  # every rank holds the whole y
        m_, s_ = (ym[d][yr - n:], ys[d][yr - n:]) if kind == gen.TOEPLITZ else (ym[d][:n], ys[d][:n])
        outs.append(hk.to_host(m_, s_))
    return outs


@pytest.mark.parametrize("kind,n,P,G", [(0, 100, 4200, 2), (1, 130, 8000, 8), (2, 77, 9000, 4),
                                        (0, 5, 17000, 8), (2, 128, 2100, 2)])
def test_coset_shards_p2p_match_oracle(hk, kind, n, P, G):
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=90 + n + G)
    want = oracle.matvec(kind, P, am, asg, xm, xsg)
    for got in sharded_p2p(hk, kind, G, am, asg, xm, xsg, P):
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("G,p2p", [(2, False), (8, True)])
def test_coset_shards_split_k2(hk, G, p2p):
    """N1 = 2^15 (n > 8192): the shard K2 runs as prepare + prepared-shard launches (MODE 1 + 4).
    Checked against the single-GPU call (itself bit-exact vs the oracle) and by fingerprints."""
    kind, n, P = 0, 8200, 4200
    assert hk.plan(kind, n, P)["log_n1"] == 15
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=8)
    got = (sharded_p2p(hk, kind, G, am, asg, xm, xsg, P)[G - 1] if p2p
           else sharded(hk, kind, G, am, asg, xm, xsg, P))
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    want = hk.to_host(*hk.matvec(kind, a, sa, x, sx, P))
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    fp.check(kind, am, asg, xm, xsg, *got)


def sharded_sliced(hk, kind, G, am, asg, xm, xsg, P, p2p=False):
    """Sliced sharding with G emulated ranks: rank g slices and row-transforms only its 1/G of the
    matrix positions (hk_hankel_shard_slice), the sigma-blocks are exchanged all-to-all, every rank
    column-transforms its block gathered from the slices (hk_hankel_shard_columns), then the coset
    exchange and K3 as in sharded() / sharded_p2p().  p2p: both exchanges fused into the stores,
    the peer pointers are the other emulated ranks' buffers."""
    n = xm.shape[0]
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    wss = [hk.ShardWorkspace(kind, n, P, G) for _ in range(G)]
    info = wss[0].info
    sw, sc = info["slice_buffer_words"], info["slice_chunk_words"]
    assert sw > 0
    chunk, rpr, yr, Ly = info["chunk_words"], info["rows_per_rank"], info["y_rows"], hk.out_limbs(P)
    if p2p:
        srecv = [torch.zeros((sw,), dtype=torch.int32, device="cuda") for _ in range(G)]
        for g in range(G):
            hk.shard_slice_p2p(wss[g], g, a, sa, x, sx, [t.data_ptr() for t in srecv])
        torch.cuda.synchronize()
        recv = [torch.full((info["buffer_words"],), -1, dtype=torch.int32, device="cuda") for _ in range(G)]
        for g in range(G):
            hk.shard_columns_p2p(wss[g], g, srecv[g], [t.data_ptr() for t in recv])
        torch.cuda.synchronize()
        ym = [torch.full((yr, Ly), -7, dtype=torch.int64, device="cuda") for _ in range(G)]
        ys = [torch.full((yr,), 9, dtype=torch.int8, device="cuda") for _ in range(G)]
        for g in range(G):
            hk.shard_finish_p2p(wss[g], g, recv[g], [t.data_ptr() for t in ym], [t.data_ptr() for t in ys])
        torch.cuda.synchronize()
        for g in range(G):
            assert wss[g].status() == hk.HK_OK
        outs = []
        for d in range(G):
            m_, s_ = (ym[d][yr - n:], ys[d][yr - n:]) if kind == gen.TOEPLITZ else (ym[d][:n], ys[d][:n])
            outs.append(hk.to_host(m_, s_))
        for o in outs[1:]:
            assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])
        return outs[0]
    ssend = [torch.zeros((sw,), dtype=torch.int32, device="cuda") for _ in range(G)]
    for g in range(G):
        hk.shard_slice(wss[g], g, a, sa, x, sx, ssend[g])
    srecv = [torch.cat([ssend[g][r * sc:(r + 1) * sc] for g in range(G)]) for r in range(G)]
    send = [torch.full((info["buffer_words"],), -1, dtype=torch.int32, device="cuda") for _ in range(G)]
    for g in range(G):
        hk.shard_columns(wss[g], g, srecv[g], send[g])
    recv = [torch.cat([send[g][r * chunk:(r + 1) * chunk] for g in range(G)]) for r in range(G)]
    y_pads = []
    for g in range(G):
        ym = torch.full((yr, Ly), -7, dtype=torch.int64, device="cuda")
        ys = torch.full((yr,), 9, dtype=torch.int8, device="cuda")
        hk.shard_finish(wss[g], g, recv[g], ym, ys)
        y_pads.append((ym, ys))
    for g in range(G):
        assert wss[g].status() == hk.HK_OK
    ym = torch.cat([y_pads[g][0][g * rpr:(g + 1) * rpr] for g in range(G)])
    ys = torch.cat([y_pads[g][1][g * rpr:(g + 1) * rpr] for g in range(G)])
    torch.cuda.synchronize()
    if kind == gen.TOEPLITZ:
        ym, ys = ym[yr - n:], ys[yr - n:]
    else:
        ym, ys = ym[:n], ys[:n]
    return hk.to_host(ym, ys)


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("kind,n,P,G", [
    (0, 100, 4200, 2), (0, 100, 4200, 8), (1, 77, 4200, 4), (1, 130, 8000, 8), (2, 64, 4200, 4),
    (2, 77, 9000, 8), (0, 40, 17000, 4), (0, 257, 2100, 2), (2, 128, 2100, 4), (1, 1000, 5000, 8)])
def test_sliced_shards_match_oracle(hk, kind, n, P, G, p2p):
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=140 + n + G)
    got = sharded_sliced(hk, kind, G, am, asg, xm, xsg, P, p2p)
    want = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_sliced_shards_carry_stress(hk):
    kind, n, P, G = 1, 96, 16608, 4
    am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=5, recipe="carry_stress")
    got = sharded_sliced(hk, kind, G, am, asg, xm, xsg, P)
    want = oracle.matvec(kind, P, am, asg, xm, xsg)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("G,p2p", [(2, False), (4, True), (8, False)])
def test_sliced_shards_c2_fingerprints(hk, G, p2p):
    c = gen.CONFIGS["C2"]
    am, asg, xm, xsg = gen.config_inputs("C2")
    ym, ys = sharded_sliced(hk, c["kind"], G, am, asg, xm, xsg, c["P"], p2p)
    fp.check(c["kind"], am, asg, xm, xsg, ym, ys)
    rows = np.arange(0, c["n"], 97)
    wm, ws = oracle.matvec(c["kind"], c["P"], am, asg, xm, xsg, rows=rows)
    assert np.array_equal(ym[rows], wm) and np.array_equal(ys[rows], ws)


@pytest.mark.parametrize("G", [2, 8])
def test_sliced_shards_c3_match_single_gpu(hk, G):
    """C3 (n = 8000, P = 33,216): the sliced shards equal the single-GPU call word for word."""
    c = gen.CONFIGS["C3"]
    am, asg, xm, xsg = gen.config_inputs("C3")
    got = sharded_sliced(hk, c["kind"], G, am, asg, xm, xsg, c["P"], p2p=(G == 8))
    a, sa = hk.to_device(am, asg)
    x, sx = hk.to_device(xm, xsg)
    want = hk.to_host(*hk.matvec(c["kind"], a, sa, x, sx, c["P"]))
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_sliced_plan_unsupported_at_n1_2p15(hk):
    """N1 = 2^15 has no sliced K2 (the column block does not fit shared memory): the plan reports
    slice_buffer_words = 0 and the slice entry points refuse with HK_EUNSUPPORTED."""
    info = hk.shard_plan(0, 8200, 4200, 4)
    assert info["slice_buffer_words"] == 0
    ws = hk.ShardWorkspace(0, 8200, 4200, 4)
    d = torch.zeros(8, dtype=torch.int32, device="cuda")
    rc = hk._lib.hk_hankel_shard_columns(0, 8200, 4200, 4, 0, d.data_ptr(), d.data_ptr(), ws.ptr,
                                         ws.nbytes, hk._stream_ptr())
    assert rc == hk.HK_EUNSUPPORTED
