"""Multi-GPU matvec, one process per GPU, torch.distributed for the plumbing.

* CosetShardedMatvec -- plan P-2 (sigma-coset sharding, the recommended plan): rank g produces
  only block g of the slice-transform outputs of every entry (coset fold inside K1), runs K2 on
  its N2/G columns per prime and writes per-destination row-block chunks; one all-to-all moves
  Y^ from column ownership to row ownership; rank g finishes its row block (K3); an all-gather of
  the equal-size y blocks gives every rank y.  Compute per rank ~1/G of K2/K3 and of K1's
  transforms (slicing is replicated).  With peer memory (torch symmetric memory over NVLink,
  the default when available) both exchanges are fused into the kernels' stores: K2 writes each
  row-block chunk straight into the destination rank's receive buffer and K3 writes its y rows
  into every rank's y; a device-side barrier follows each phase.  Otherwise NCCL
  all_to_all_single / all_gather_into_tensor do the exchanges.
* ShardedHankel -- plan P-3, north_star's literal row-block sharding (below).

One process per GPU (torchrun), torch.distributed for the plumbing (NCCL over NVLink on GPUs,
gloo in the CPU tests).  Rank g owns output rows [r0, r0 + nr) of the n x n Hankel product; its
shard is itself a Hankel product -- the nr x n window over a[r0 .. r0 + nr + n - 2] (PAPER.md
P:50-60: row i only touches a_i .. a_{i+n-1}) -- computed by the C-ABI CUDA path
(hk_hankel_rect_matvec).  The y rows are then all-gathered so every rank holds the full y.
There is no other data-path exchange.

The per-shard compute is a parameter so the sharding / gather logic can be exercised on CPU
(gloo) with any exact shard function; the default is the CUDA path.
"""
from __future__ import annotations

import os

import numpy as np


def row_blocks(n: int, G: int) -> list[tuple[int, int]]:
    """Balanced contiguous row blocks (r0, nr) for G ranks; the first n % G get one extra row."""
    if G < 1 or n < 1:
        raise ValueError("need n >= 1 and G >= 1")
    base, extra = divmod(n, G)
    out, r0 = [], 0
    for g in range(G):
        nr = base + (1 if g < extra else 0)
        out.append((r0, nr))
        r0 += nr
    return out


def window(a_mag, a_sign, r0: int, nr: int, n: int):
    """Entries a[r0 .. r0 + nr + n - 2] (0-based) feeding output rows r0 .. r0 + nr - 1."""
    return a_mag[r0:r0 + nr + n - 1], a_sign[r0:r0 + nr + n - 1]


def _cuda_shard(a_mag, a_sign, x_mag, x_sign, P, m, out=None, ws=None):
    from . import hankel_rect_matvec
    return hankel_rect_matvec(a_mag, a_sign, x_mag, x_sign, P, m, out=out, ws=ws, check=False)


class ShardedHankel:
    """Prepared sharded problem for repeated steps (bench): owns this rank's window, its
    workspace, the local y block and the gathered y."""

    def __init__(self, a_mag, a_sign, x_mag, x_sign, P, group=None, compute=None):
        import torch
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = int(x_mag.shape[0])
        self.P = int(P)
        self.blocks = row_blocks(self.n, self.G)
        self.r0, self.nr = self.blocks[self.rank]
        self.nr_max = max(nr for _, nr in self.blocks)
        # own copies of the window: a view would start r0 L 8 bytes into a_mag, which is only
        # 8-byte aligned when r0 L is odd, and the C ABI needs 16-byte-aligned magnitudes
        self.win = tuple(t.clone() for t in window(a_mag, a_sign, self.r0, self.nr, self.n))
        self.x = (x_mag, x_sign)
        self.compute = compute or _cuda_shard
        Ly = 2 * ((P + 63) // 64) + 1
        dev = a_mag.device
        self.ws = None
        if compute is None and self.nr > 0:
            from . import Workspace, HANKEL
            self.ws = Workspace(HANKEL, self.n, self.P, m=self.nr)
        # local block padded to nr_max rows so every rank contributes an equal-size chunk
        self.y_loc = torch.zeros((self.nr_max, Ly), dtype=a_mag.dtype, device=dev)
        self.s_loc = torch.zeros((self.nr_max,), dtype=torch.int8, device=dev)
        self.y_all = torch.empty((self.G * self.nr_max, Ly), dtype=a_mag.dtype, device=dev)
        self.s_all = torch.empty((self.G * self.nr_max,), dtype=torch.int8, device=dev)

    def check_status(self):
        """MIN all-reduce of every rank's data status (HK_OK = 0, errors < 0): raises HKError on
        every rank if any rank's inputs were rejected (its y rows are then unspecified)."""
        _agree_status(self.dist, self.group, self.ws, self.x[0].device)

    def step(self, check=False):
        if self.nr > 0:
            kw = {"ws": self.ws} if self.ws is not None else {}
            out = (self.y_loc[: self.nr], self.s_loc[: self.nr])
            ym, ys = self.compute(self.win[0], self.win[1], self.x[0], self.x[1], self.P, self.nr,
                                  out=out, **kw)
            if ym.data_ptr() != self.y_loc.data_ptr():
                self.y_loc[: self.nr].copy_(ym)
                self.s_loc[: self.nr].copy_(ys)
        if check:
            self.check_status()
        self._gather()
        return self.result()

    def _gather(self):
        d = self.dist
        try:
            d.all_gather_into_tensor(self.y_all, self.y_loc, group=self.group)
            d.all_gather_into_tensor(self.s_all, self.s_loc, group=self.group)
        except (RuntimeError, NotImplementedError, AttributeError):  # backends without _allgather_base
            ys = list(self.y_all.chunk(self.G))
            ss = list(self.s_all.chunk(self.G))
            d.all_gather(ys, self.y_loc, group=self.group)
            d.all_gather(ss, self.s_loc, group=self.group)

    def result(self):
        """Full y (n rows) in row order, from the gathered padded blocks."""
        import torch
        idx = np.concatenate([np.arange(g * self.nr_max, g * self.nr_max + nr)
                              for g, (_, nr) in enumerate(self.blocks)])
        it = torch.from_numpy(idx).to(self.y_all.device)
        return self.y_all.index_select(0, it), self.s_all.index_select(0, it)


def _agree_status(dist, group, ws, device):
    import torch
    from . import HK_OK, HKError
    code = ws.status() if ws is not None else HK_OK
    t = torch.tensor([code], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    worst = int(t.item())
    if worst != HK_OK:
        raise HKError(worst, "sharded matvec data status (MIN over ranks)")


def hankel_matvec(a_mag, a_sign, x_mag, x_sign, P, group=None, compute=None, check=True):
    """y = A_H x sharded by rows over the process group; returns the full y on every rank."""
    return ShardedHankel(a_mag, a_sign, x_mag, x_sign, P, group=group, compute=compute).step(check)


# ---------------------------------------------------------------------------------------------
# plan P-2: sigma-coset sharding
def _cuda_forward(ws, g, a_mag, a_sign, x_mag, x_sign, send):
    from . import shard_forward
    shard_forward(ws, g, a_mag, a_sign, x_mag, x_sign, send)


def _cuda_finish(ws, g, recv, y_mag, y_sign):
    from . import shard_finish
    shard_finish(ws, g, recv, y_mag, y_sign)


def _cuda_slice(ws, g, a_mag, a_sign, x_mag, x_sign, slice_send):
    from . import shard_slice
    shard_slice(ws, g, a_mag, a_sign, x_mag, x_sign, slice_send)


def _cuda_columns(ws, g, slice_recv, send):
    from . import shard_columns
    shard_columns(ws, g, slice_recv, send)


def _want_sliced(sliced, info, G) -> bool:
    """Sliced sharding (each rank slices 1/G of the positions) when the plan supports it: by
    default from G = 4 on, where the replicated slicing of the coset mode costs more than the
    extra slice exchange (profiles/r02/shard_phase_times_C3.json); HK_SLICED=0/1 overrides."""
    ok = int(info.get("slice_buffer_words", 0)) > 0
    env = os.environ.get("HK_SLICED")
    if env is not None:
        return env == "1" and ok
    if sliced == "auto":
        return G >= 4 and ok
    if sliced and not ok:
        raise ValueError("sliced sharding unsupported for this plan (N1 > 2^14 or too few positions)")
    return bool(sliced)


class CosetShardedMatvec:
    """Prepared sigma-coset-sharded problem (kind in {Hankel, Toeplitz, circulant}, n x n) for
    repeated steps: rank-local workspace, all-to-all send / receive buffers and the padded y.

    ``forward(ws, g, a, sa, x, sx, send)`` and ``finish(ws, g, recv, y, s)`` default to the CUDA
    phases (hk_hankel_shard_forward / _finish); tests inject stand-ins to exercise the exchange
    on CPU (gloo), with ``info`` the layout (paper_1402_5287_b200.shard_plan).

    ``sliced``: the forward phase runs as slice -> slice all-to-all -> columns
    (hk_hankel_shard_slice / _columns, stand-ins ``slice(ws, g, a, sa, x, sx, slice_send)`` and
    ``columns(ws, g, slice_recv, send)``): rank g slices and row-transforms only positions
    [g Rs, (g+1) Rs) of a and x, and gathers its sigma-block from every rank's slices."""

    def __init__(self, kind, a_mag, a_sign, x_mag, x_sign, P, group=None, forward=None,
                 finish=None, info=None, p2p="auto", sliced="auto", slice=None, columns=None):
        import torch
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.kind, self.P = int(kind), int(P)
        self.n = int(x_mag.shape[0])
        self.inputs = (a_mag, a_sign, x_mag, x_sign)
        dev = a_mag.device
        self.ws = None
        if forward is None or finish is None:
            from . import ShardWorkspace
            self.ws = ShardWorkspace(kind, self.n, P, self.G, device=dev)
            info = self.ws.info
        self.info = info
        self.forward = forward or _cuda_forward
        self.finish = finish or _cuda_finish
        injected = forward is not None or finish is not None
        self.slice_fn = slice or (None if injected else _cuda_slice)
        self.columns_fn = columns or (None if injected else _cuda_columns)
        if self.slice_fn is None or self.columns_fn is None:
            sliced = False
        self.sliced = _want_sliced(sliced, info, self.G) if sliced else False
        words, rpr, yr = info["buffer_words"], info["rows_per_rank"], info["y_rows"]
        self.rpr, self.y_rows = int(rpr), int(yr)
        self.slice_words = int(info.get("slice_buffer_words", 0)) if self.sliced else 0
        Ly = 2 * ((P + 63) // 64) + 1
        self.p2p = False
        if os.environ.get("HK_P2P", "1") == "0":
            p2p = False
        if p2p and self.ws is not None and self.G > 1:
            # every rank takes the same decision: setup steps are agreed on with MIN all-reduces,
            # so a rank that cannot map peer memory never leaves the others in a rendezvous
            self.p2p = self._setup_p2p(words, yr, Ly, a_mag.dtype, dev)
            if not self.p2p and p2p != "auto":
                raise RuntimeError("peer-memory exchange requested but unavailable")
        if not self.p2p:
            self.send = torch.zeros((words,), dtype=torch.int32, device=dev)
            self.recv = torch.zeros((words,), dtype=torch.int32, device=dev)
            self.y_pad = torch.zeros((yr, Ly), dtype=a_mag.dtype, device=dev)
            self.s_pad = torch.zeros((yr,), dtype=torch.int8, device=dev)
            if self.sliced:  # zero once: positions no rank owns (past the last entry) stay zero
                self.slice_send = torch.zeros((self.slice_words,), dtype=torch.int32, device=dev)
                self.slice_recv = torch.zeros((self.slice_words,), dtype=torch.int32, device=dev)

    def _agree(self, ok: bool, dev) -> bool:
        import torch
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())

    def _setup_p2p(self, words, yr, Ly, mag_dtype, dev) -> bool:
        """Receive buffer and padded y in torch symmetric memory (NVLink peer-mapped): the
        all-to-all is fused into K2's stores and the y all-gather into K3's stores."""
        import torch
        try:
            import torch.distributed._symmetric_memory as symm_mem
            bufs = [symm_mem.empty(words, dtype=torch.int32, device=dev),
                    symm_mem.empty(yr, Ly, dtype=mag_dtype, device=dev),
                    symm_mem.empty(yr, dtype=torch.int8, device=dev)]
            if self.sliced:
                bufs.append(symm_mem.empty(self.slice_words, dtype=torch.int32, device=dev))
                bufs[-1].zero_()  # positions no rank owns stay zero (K2 reads them)
            ok = True
        except Exception:
            ok = False
        if not self._agree(ok, dev):
            return False
        try:
            grp = self.group if self.group is not None else self.dist.group.WORLD
            handles = [symm_mem.rendezvous(t, grp) for t in bufs]

            def peer_ptrs(t, h):
                off = t.data_ptr() - int(h.buffer_ptrs[self.rank])
                return [int(p) + off for p in h.buffer_ptrs]

            ptrs = [peer_ptrs(t, h) for t, h in zip(bufs, handles)]
            ok = all(len(p) == self.G and all(p) for p in ptrs)
        except Exception:
            ok = False
        if not self._agree(ok, dev):
            return False
        self.recv, self.y_pad, self.s_pad = bufs[:3]
        self.recv_ptrs, self.y_ptrs, self.s_ptrs = ptrs[:3]
        self.h_recv, self.h_y = handles[0], handles[1]
        if self.sliced:
            self.slice_recv, self.slice_ptrs, self.h_slice = bufs[3], ptrs[3], handles[3]
            handles[3].barrier()  # every rank's zero-fill is done before any peer stores into it
        return True

    def compute_slice(self):
        """Sliced phase 1a: K1 over this rank's positions, sigma-blocks scattered by destination."""
        if self.p2p:
            from . import shard_slice_p2p
            shard_slice_p2p(self.ws, self.rank, *self.inputs, self.slice_ptrs)
        else:
            self.slice_fn(self.ws, self.rank, *self.inputs, self.slice_send)

    def exchange_slices(self):
        if self.p2p:  # every rank's K1 stores into this rank's slice buffer are done
            self.h_slice.barrier()
        else:
            self.dist.all_to_all_single(self.slice_recv, self.slice_send, group=self.group)

    def compute_columns(self):
        """Sliced phase 1b: K2 on this rank's sigma-block, gathered from the received slices."""
        if self.p2p:
            from . import shard_columns_p2p
            shard_columns_p2p(self.ws, self.rank, self.slice_recv, self.recv_ptrs)
        else:
            self.columns_fn(self.ws, self.rank, self.slice_recv, self.send)

    def compute_forward(self):
        if self.sliced:
            self.compute_slice()
            self.exchange_slices()
            self.compute_columns()
        elif self.p2p:
            from . import shard_forward_p2p
            shard_forward_p2p(self.ws, self.rank, *self.inputs, self.recv_ptrs)
        else:
            self.forward(self.ws, self.rank, *self.inputs, self.send)

    def exchange(self):
        if self.p2p:  # every rank's K2 stores into this rank's receive buffer are done
            self.h_recv.barrier()
        else:
            self.dist.all_to_all_single(self.recv, self.send, group=self.group)

    def compute_finish(self):
        if self.p2p:
            from . import shard_finish_p2p
            shard_finish_p2p(self.ws, self.rank, self.recv, self.y_ptrs, self.s_ptrs)
        else:
            self.finish(self.ws, self.rank, self.recv, self.y_pad, self.s_pad)

    def gather(self):
        if self.p2p:  # every rank's K3 stores into this rank's y are done
            self.h_y.barrier()
            return
        r0, r1 = self.rank * self.rpr, (self.rank + 1) * self.rpr
        d = self.dist
        try:  # in place: this rank's block already sits in its slot of the output
            d.all_gather_into_tensor(self.y_pad, self.y_pad[r0:r1], group=self.group)
            d.all_gather_into_tensor(self.s_pad, self.s_pad[r0:r1], group=self.group)
        except (RuntimeError, NotImplementedError, AttributeError):  # backends without it
            ym, ys = self.y_pad[r0:r1].clone(), self.s_pad[r0:r1].clone()
            d.all_gather(list(self.y_pad.chunk(self.G)), ym, group=self.group)
            d.all_gather(list(self.s_pad.chunk(self.G)), ys, group=self.group)

    def result(self):
        """The final y (views of the padded buffer): rows [0, n), or the last n for Toeplitz."""
        if self.kind == 1:  # Toeplitz: reversed rows are padded at the front
            return self.y_pad[self.y_rows - self.n:], self.s_pad[self.y_rows - self.n:]
        return self.y_pad[: self.n], self.s_pad[: self.n]

    def check_status(self):
        """MIN all-reduce of every rank's data status; raises HKError on every rank if any rank's
        K1 rejected its inputs."""
        _agree_status(self.dist, self.group, self.ws, self.inputs[0].device)

    def step(self, check=False):
        self.compute_forward()
        if check:
            self.check_status()
        self.exchange()
        self.compute_finish()
        self.gather()
        return self.result()


def coset_matvec(kind, a_mag, a_sign, x_mag, x_sign, P, group=None, check=True):
    """y = A x over the process group with plan P-2; returns the full y on every rank."""
    return CosetShardedMatvec(kind, a_mag, a_sign, x_mag, x_sign, P, group=group).step(check)


class CosetStream:
    """Throughput mode of plan P-2 (the multi-GPU rate of a stream of independent
    matvecs, the paper's repeated-product use P:32-36).  ``slots`` CosetShardedMatvec
    instances (each with its own workspace, exchange buffers and padded y) are used round-robin.
    On CUDA the exchanges -- the all-to-all (or, with peer memory, the device barrier that ends
    the fused K2 stores) and the y all-gather (or the barrier after K3's fused stores) -- are
    enqueued on a communication stream, so matvec t's exchanges overlap the K1/K2 of matvec t+1
    and the K3 of matvec t-1 on the compute stream.  The collectives are issued in the same
    order on every rank (X0, X1, G0, X2, G1, ...), which NCCL requires.

    Slot reuse: matvec t (slot t mod S) starts only after the y all-gather of matvec t - S has
    completed on this rank; that all-gather (NCCL) or barrier (peer memory) also proves every
    rank finished reading its receive buffer of that slot, so K2's stores of matvec t -- local or
    into peers -- cannot overwrite data still in use.  With peer memory and a ``consume``
    callback, one more barrier after ``consume`` keeps other ranks' K3 stores of matvec t + S out
    of this rank's y until it has been consumed.

    Sliced slots add a third exchange per matvec: iteration t issues, in this order, the finish of
    t - 2 (K3, y all-gather), the slicing of t (K1) and its slice all-to-all, then the columns of
    t - 1 (K2) and its coset all-to-all -- communication order GA(t-2), XS(t), XC(t-1) on every
    rank, and the compute stream runs K3(t-2), K1(t), K2(t-1) while the exchanges of the
    neighbouring matvecs are in flight.  The slot-reuse argument above holds unchanged: K1 of
    matvec t (which with peer memory stores into the peers' slice buffers) waits for the
    all-gather / barrier of t - S, issued earlier in the same iteration for S = 2.

    The CPU (gloo) path runs the same sequence synchronously, for the tests."""

    def __init__(self, kind, inputs_like, P, slots=3, group=None, forward=None, finish=None,
                 info=None, p2p="auto", sliced="auto", slice=None, columns=None):
        import torch
        if slots < 2:
            raise ValueError("CosetStream needs at least 2 slots (slot reuse waits on matvec t - S)")
        self.slots = [CosetShardedMatvec(kind, *inputs_like, P, group=group, forward=forward,
                                         finish=finish, info=info, p2p=p2p, sliced=sliced,
                                         slice=slice, columns=columns) for _ in range(slots)]
        self.S = len(self.slots)
        self.cuda = inputs_like[0].is_cuda
        self.p2p = self.slots[0].p2p
        self.sliced = self.slots[0].sliced
        self.comp = self.comm = None
        if self.cuda:
            self.comp = torch.cuda.current_stream()
            self.comm = torch.cuda.Stream(device=inputs_like[0].device)
            ev = lambda: [torch.cuda.Event() for _ in range(self.S)]  # noqa: E731
            self.ev_fwd, self.ev_x, self.ev_fin, self.ev_done = ev(), ev(), ev(), ev()
            self.ev_a, self.ev_xs = ev(), ev()

    def _stream(self, s):
        import contextlib
        import torch
        return torch.cuda.stream(s) if self.cuda else contextlib.nullcontext()

    def run(self, problems, consume=None, check=False):
        """Runs y_t = A_t x_t for every (a_mag, a_sign, x_mag, x_sign) in ``problems``; calls
        ``consume(t, y_mag, y_sign)`` (on the communication stream when CUDA) once y_t is complete
        on this rank -- the views stay valid only until slot t mod S is reused.  ``check``: the
        data status of every matvec is captured on the device and MIN-all-reduced at the end
        (HKError on every rank if any rank rejected an input).  Returns the number of matvecs."""
        import torch
        S, used = self.S, [False] * self.S
        statuses = []

        def finish(t):
            s = t % S
            sl = self.slots[s]
            with self._stream(self.comp):
                if self.cuda:
                    self.comp.wait_event(self.ev_x[s])
                sl.compute_finish()
                if self.cuda:
                    self.ev_fin[s].record(self.comp)
            with self._stream(self.comm):
                if self.cuda:
                    self.comm.wait_event(self.ev_fin[s])
                sl.gather()
                if consume is not None:
                    consume(t, *sl.result())
                    if self.p2p:
                        sl.h_y.barrier()
                if self.cuda:
                    self.ev_done[s].record(self.comm)

        def status(sl, prob):
            if check and sl.ws is not None:
                w = torch.empty((1,), dtype=torch.int32, device=prob[0].device)
                w.copy_(sl.ws.status_word())
                statuses.append(w)

        count = 0
        if self.sliced:
            count = self._run_sliced(problems, finish, status, used)
            problems = ()
        for t, prob in enumerate(problems):
            s = t % S
            sl = self.slots[s]
            with self._stream(self.comp):
                if self.cuda and used[s]:
                    self.comp.wait_event(self.ev_done[s])
                sl.inputs = tuple(prob)
                sl.compute_forward()
                status(sl, prob)
                if self.cuda:
                    self.ev_fwd[s].record(self.comp)
            used[s] = True
            with self._stream(self.comm):
                if self.cuda:
                    self.comm.wait_event(self.ev_fwd[s])
                sl.exchange()
                if self.cuda:
                    self.ev_x[s].record(self.comm)
            if t >= 1:
                finish(t - 1)
            count += 1
        if count and not self.sliced:
            finish(count - 1)
        if self.cuda:
            self.comp.wait_stream(self.comm)
        if check:
            from . import HK_OK, HKError
            worst = torch.stack(statuses).min().reshape(1) if statuses else torch.zeros(
                (1,), dtype=torch.int32, device=self.slots[0].inputs[0].device)
            sl = self.slots[0]
            sl.dist.all_reduce(worst, op=sl.dist.ReduceOp.MIN, group=sl.group)
            if int(worst.item()) != HK_OK:
                raise HKError(int(worst.item()), "coset stream data status (MIN over ranks)")
        return count

    def _run_sliced(self, problems, finish, status, used):
        S = self.S

        def columns(t):
            s = t % S
            sl = self.slots[s]
            with self._stream(self.comp):
                if self.cuda:
                    self.comp.wait_event(self.ev_xs[s])
                sl.compute_columns()
                if self.cuda:
                    self.ev_fwd[s].record(self.comp)
            with self._stream(self.comm):
                if self.cuda:
                    self.comm.wait_event(self.ev_fwd[s])
                sl.exchange()
                if self.cuda:
                    self.ev_x[s].record(self.comm)

        count = 0
        for t, prob in enumerate(problems):
            s = t % S
            sl = self.slots[s]
            if t >= 2:
                finish(t - 2)
            with self._stream(self.comp):
                if self.cuda and used[s]:
                    self.comp.wait_event(self.ev_done[s])
                sl.inputs = tuple(prob)
                sl.compute_slice()
                status(sl, prob)
                if self.cuda:
                    self.ev_a[s].record(self.comp)
            used[s] = True
            with self._stream(self.comm):
                if self.cuda:
                    self.comm.wait_event(self.ev_a[s])
                sl.exchange_slices()
                if self.cuda:
                    self.ev_xs[s].record(self.comm)
            if t >= 1:
                columns(t - 1)
            count += 1
        if count:
            columns(count - 1)
            if count >= 2:
                finish(count - 2)
            finish(count - 1)
        return count
