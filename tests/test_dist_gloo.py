"""Multi-process (world_size 2, gloo, CPU) test of the row-block sharding + all-gather path of
paper_1402_5287_b200.dist.  The per-shard compute is the oracle here (tests may call it); on
GPUs the same ShardedHankel runs the CUDA shard kernel over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hkinputs as gen
import oracle
from paper_1402_5287_b200 import dist as hkdist


def test_row_blocks_cover_rows_exactly():
    for n in (1, 2, 7, 8000, 16384):
        for G in (1, 2, 3, 4, 8):
            b = hkdist.row_blocks(n, G)
            assert len(b) == G and sum(nr for _, nr in b) == n
            assert all(b[i][0] + b[i][1] == b[i + 1][0] for i in range(G - 1))
            assert max(nr for _, nr in b) - min(nr for _, nr in b) <= 1


def test_window_is_a_hankel_shard():
    """Rows r0..r0+nr-1 of the n x n Hankel product == the nr x n window product."""
    P, n = 300, 11
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=5)
    full = oracle.matvec(0, P, am, asg, xm, xsg, threads=2)
    for r0, nr in hkdist.row_blocks(n, 3):
        wm, ws = hkdist.window(am, asg, r0, nr, n)
        part = oracle.matvec(0, P, wm, ws, xm, xsg, m=nr, threads=2)
        assert np.array_equal(part[0], full[0][r0:r0 + nr])
        assert np.array_equal(part[1], full[1][r0:r0 + nr])


def _oracle_shard(a_mag, a_sign, x_mag, x_sign, P, m, out=None):
    ym, ys = oracle.matvec(0, P, a_mag.numpy().view(np.uint64), a_sign.numpy(),
                           x_mag.numpy().view(np.uint64), x_sign.numpy(), m=m, threads=1)
    return torch.from_numpy(ym.view(np.int64)), torch.from_numpy(ys)


def _worker(rank, world, port, n, P, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=17)
        t = [torch.from_numpy(am.view(np.int64)), torch.from_numpy(asg),
             torch.from_numpy(xm.view(np.int64)), torch.from_numpy(xsg)]
        ym, ys = hkdist.hankel_matvec(*t, P, compute=_oracle_shard)
        q.put((rank, ym.numpy().view(np.uint64).copy(), ys.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [9, 16])
def test_sharded_matvec_gloo_world2(n):
    P = 400
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, P, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    am, asg, xm, xsg = gen.make_inputs(0, n, P, seed=17)
    wm, ws = oracle.matvec(0, P, am, asg, xm, xsg, threads=2)
    for _, ym, ys in res:
        assert np.array_equal(ym, wm) and np.array_equal(ys, ws)


# ---------------------------------------------------------------------------------------------
# plan P-2 (sigma-coset sharding): exchange and gather logic of CosetShardedMatvec on CPU.
# The CUDA phases are replaced by stand-ins that write / check labelled words, so the test pins
# the all-to-all chunk routing, the in-place all-gather of the padded y, and the Toeplitz layout.
def _label(src, dst, j):
    return (src * 7919 + dst * 104729 + j) % (2 ** 31 - 1)


def _coset_worker(rank, world, port, kind, n, P, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1402_5287_b200 as hk
        info = hk.shard_plan(kind, n, P, world)  # host-side planner, no GPU needed
        chunk, rpr = info["chunk_words"], info["rows_per_rank"]
        j = torch.arange(chunk, dtype=torch.int64)

        def forward(ws, g, am, asg, xm, xsg, send):
            for dst in range(world):
                send[dst * chunk:(dst + 1) * chunk] = torch.tensor(
                    [_label(g, dst, int(v)) for v in j[:3]] + [0] * (chunk - 3), dtype=torch.int32)

        seen = {}

        def finish(ws, g, recv, y_mag, y_sign):
            for src in range(world):
                seen[src] = [int(v) for v in recv[src * chunk:src * chunk + 3]]
            y_mag[g * rpr:(g + 1) * rpr] = 1000 + g
            y_sign[g * rpr:(g + 1) * rpr] = g + 1

        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=1)
        t = [torch.from_numpy(am.view(np.int64)), torch.from_numpy(asg),
             torch.from_numpy(xm.view(np.int64)), torch.from_numpy(xsg)]
        from paper_1402_5287_b200 import dist as hd
        sh = hd.CosetShardedMatvec(kind, *t, P, forward=forward, finish=finish, info=info)
        ym, ys = sh.step()
        q.put((rank, seen, sh.y_pad.numpy().copy(), sh.s_pad.numpy().copy(), ym.shape[0],
               int(ym[0, 0]), int(ym[-1, 0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,P", [(0, 101, 4200), (1, 101, 4200), (2, 64, 4200)])
def test_coset_exchange_gloo_world2(kind, n, P):
    import paper_1402_5287_b200 as hk
    world = 2
    info = hk.shard_plan(kind, n, P, world)
    rpr, yr = info["rows_per_rank"], info["y_rows"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coset_worker, args=(r, world, port, kind, n, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, seen, y_pad, s_pad, nrows, first, last in res:
        # all-to-all: chunk src of rank r's receive buffer is chunk r of rank src's send buffer
        for src in range(world):
            assert seen[src] == [_label(src, rank, v) for v in range(3)]
        # all-gather: block g of the padded y comes from rank g, on every rank
        for g in range(world):
            assert (y_pad[g * rpr:(g + 1) * rpr] == 1000 + g).all()
            assert (s_pad[g * rpr:(g + 1) * rpr] == g + 1).all()
        assert nrows == n and yr >= n
        if kind == 1:  # Toeplitz: final rows are the LAST n rows of the padded buffer
            assert last == 1000 + world - 1 and first == 1000 + (yr - n) // rpr
        else:
            assert first == 1000 and last == 1000 + (n - 1) // rpr


# ---------------------------------------------------------------------------------------------
# throughput mode (CosetStream): a stream of independent matvecs over S slots.  Stand-in phases
# tag every word with the problem id, so the test pins that each consumed y holds the blocks of
# its own problem from every rank, in order, across slot reuse.
def _stream_worker(rank, world, port, kind, n, P, nprob, slots, q, sliced=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1402_5287_b200 as hk
        from paper_1402_5287_b200 import dist as hd
        info = hk.shard_plan(kind, n, P, world)
        chunk, rpr = info["chunk_words"], info["rows_per_rank"]

        def forward(ws, g, am, asg, xm, xsg, send):
            pid = int(am[0, 0])
            for dst in range(world):
                send[dst * chunk:(dst + 1) * chunk] = pid * 100 + g * 10 + dst

        def finish(ws, g, recv, y_mag, y_sign):
            pids = {int(recv[src * chunk]) // 100 for src in range(world)}
            assert len(pids) == 1, pids  # every source rank's chunk is from the same problem
            routed = [int(recv[src * chunk]) % 100 for src in range(world)]
            assert routed == [src * 10 + g for src in range(world)], routed
            y_mag[g * rpr:(g + 1) * rpr] = pids.pop() * 1000 + g

        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=1)
        base = [torch.from_numpy(am.view(np.int64)), torch.from_numpy(asg),
                torch.from_numpy(xm.view(np.int64)), torch.from_numpy(xsg)]
        probs = []
        for t in range(nprob):
            a_t = base[0].clone()
            a_t[0, 0] = 7 + t  # problem id
            probs.append((a_t, base[1], base[2], base[3]))
        got = []

        def consume(t, ym, ys):
            got.append((t, [int(ym[0, 0]), int(ym[-1, 0])],
                        sorted({int(v) for v in sh.slots[t % slots].y_pad[:, 0]})))

        kw = {}
        if sliced:  # slice stand-in tags (problem, source, destination); columns checks the routing
            sc = info["slice_chunk_words"]

            def slice_(ws, g, am, asg, xm, xsg, slice_send):
                pid = int(am[0, 0])
                for dst in range(world):
                    slice_send[dst * sc:(dst + 1) * sc] = pid * 100 + g * 10 + dst

            def columns(ws, g, slice_recv, send):
                pids = {int(slice_recv[src * sc]) // 100 for src in range(world)}
                assert len(pids) == 1, pids
                routed = [int(slice_recv[src * sc]) % 100 for src in range(world)]
                assert routed == [src * 10 + g for src in range(world)], routed
                pid = pids.pop()
                for dst in range(world):
                    send[dst * chunk:(dst + 1) * chunk] = pid * 100 + g * 10 + dst

            kw = dict(sliced=True, slice=slice_, columns=columns)
        sh = hd.CosetStream(kind, base, P, slots=slots, forward=forward, finish=finish, info=info, **kw)
        assert sh.sliced == sliced
        cnt = sh.run(probs, consume=consume)
        q.put((rank, cnt, got, rpr, info["y_rows"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,slots,sliced", [(0, 3, False), (1, 2, False), (2, 3, False),
                                               (0, 2, True), (1, 3, True), (2, 2, True)])
def test_coset_stream_gloo_world2(kind, slots, sliced):
    """Sliced: the slice all-to-all, the coset all-to-all and the y all-gather of 7 problems
    interleave over 2-3 slots; every phase sees only its own problem's words, correctly routed."""
    world, n, P, nprob = 2, 64, 4200, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stream_worker,
                         args=(r, world, port, kind, n, P, nprob, slots, q, sliced))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, cnt, got, rpr, yr in res:
        assert cnt == nprob and [t for t, _, _ in got] == list(range(nprob))
        for t, _, vals in got:
            pid = 7 + t
            assert vals == [pid * 1000 + g for g in range(world)], (t, vals)


# ---------------------------------------------------------------------------------------------
# peer-memory set-up agreement: a rank that cannot allocate symmetric memory makes every rank
# fall back to the NCCL exchanges (MIN all-reduce), without a rank entering the rendezvous alone
def _p2p_fallback_worker(rank, world, port, fail_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch.distributed._symmetric_memory as symm_mem
        import paper_1402_5287_b200 as hk
        from paper_1402_5287_b200 import dist as hd
        kind, n, P = 0, 64, 4200
        info = hk.shard_plan(kind, n, P, world)
        am, asg, xm, xsg = gen.make_inputs(kind, n, P, seed=1)
        t = [torch.from_numpy(am.view(np.int64)), torch.from_numpy(asg),
             torch.from_numpy(xm.view(np.int64)), torch.from_numpy(xsg)]
        sh = hd.CosetShardedMatvec(kind, *t, P, forward=lambda *a: None, finish=lambda *a: None,
                                   info=info)
        calls = []
        if rank == fail_rank:
            def empty(*a, **k):
                raise RuntimeError("no symmetric memory here")
        else:
            def empty(*shape, dtype=None, device=None):
                return torch.zeros(shape, dtype=dtype)
        orig_e, orig_r = symm_mem.empty, symm_mem.rendezvous
        symm_mem.empty = empty
        symm_mem.rendezvous = lambda *a, **k: calls.append(1)
        try:
            ok = sh._setup_p2p(info["buffer_words"], info["y_rows"], 9, torch.int64,
                               torch.device("cpu"))
        finally:
            symm_mem.empty, symm_mem.rendezvous = orig_e, orig_r
        q.put((rank, ok, len(calls)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [0, 1])
def test_p2p_setup_falls_back_together(fail_rank):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_fallback_worker, args=(r, world, port, fail_rank, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, rendezvous_calls in res:
        assert ok is False and rendezvous_calls == 0


def test_sliced_mode_selection(monkeypatch):
    """Auto: sliced from G = 4 on when the plan supports it; HK_SLICED=0/1 overrides; an explicit
    request the plan cannot serve raises."""
    from paper_1402_5287_b200.dist import _want_sliced
    ok, no = {"slice_buffer_words": 10}, {"slice_buffer_words": 0}
    monkeypatch.delenv("HK_SLICED", raising=False)
    assert [_want_sliced("auto", ok, G) for G in (2, 4, 8)] == [False, True, True]
    assert _want_sliced("auto", no, 8) is False
    assert _want_sliced(True, ok, 2) is True
    with pytest.raises(ValueError):
        _want_sliced(True, no, 4)
    monkeypatch.setenv("HK_SLICED", "0")
    assert _want_sliced("auto", ok, 8) is False
    monkeypatch.setenv("HK_SLICED", "1")
    assert _want_sliced("auto", ok, 2) is True and _want_sliced("auto", no, 2) is False
