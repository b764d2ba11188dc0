"""Multi-GPU factorization and solve: one process per GPU, torch.distributed.

Layout (BASELINE.json north_star): the m x n matrix is split 1D block-cyclic
by column blocks of width bw (nb, or 2 nb = a panel pair on the GPU) -- block
k lives on rank k % G as local block k // G, local blocks stored contiguously
(column-major, leading dim lda).

Factorization, step k (j0 = k bw, m_k = m - j0):
  1. the owner factors block k in place (qrb_op_panel_block: one or two
     nb-wide panels + the merged block reflector T2);
  2. the owner packs (V_k, T2_k, tau_k) into one contiguous buffer and
     broadcasts it (NCCL over NVLink/NVSwitch on the GPU box; gloo in the CPU
     tests) -- the single exchange of the step;
  3. every rank applies Q_k^T to its local blocks with index > k
     (qrb_op_apply_qt: the DMMA trailing update, K = bw).
With look-ahead the owner of block k+1 updates that block first, then factors
and broadcasts it on a second stream while its own remaining update runs on
capped GEMM grids (qrb_op_apply_qt_begin / _cols, "grid_cap") -- the
single-GPU schedule of qrb_api.cu right_looking, per rank.
The reference has no distributed code; its analogue of
scaling past one device is the out-of-core tile schedule (task_engine.py:187-217).

Solve: slices are independent, so after the factorization the factored
panels and the T factors are all-gathered once and every rank solves its
share of the slices against a full resident copy (no communication during
the solve).

The per-step local arithmetic is injected (``ops``): the product uses
:class:`CudaOps` (the sm_100a library); the CPU tests inject numpy ops to check
the distributed schedule itself over gloo.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import SingularMatrixError


def owner_of(k: int, world: int) -> int:
    return k % world


def local_panels(nblocks: int, rank: int, world: int) -> list[int]:
    """Global indices of the column blocks rank owns, in local storage order."""
    return list(range(rank, nblocks, world))


def local_cols(n: int, bw: int, rank: int, world: int) -> int:
    nblk = -(-n // bw)
    return sum(min(bw, n - k * bw) for k in local_panels(nblk, rank, world))


def first_local_after(k: int, rank: int, world: int) -> int:
    """Local block index of the first owned block with global index > k."""
    if rank > k:
        return 0
    return (k - rank) // world + 1


def panel_home(k: int, nb: int, bw: int, world: int) -> tuple[int, int]:
    """(owner rank, local column) of the nb-wide panel k in a bw-block layout."""
    j0 = k * nb
    blk = j0 // bw
    return owner_of(blk, world), (blk // world) * bw + (j0 - blk * bw)


def owner_chain_sms(mk: int, rest: int, w: int, m_next: int, nb: int, sms: int = 148,
                    r_min: int = 24, lat_ms: float = 0.25, rate: float = 34.0e9) -> int:
    """SMs left to the owner's next-block chain while its trailing update (rest
    columns, K = w, m_k rows) runs capped on the others: the R in
    {r_min, 32, 48, 64, 96} minimising max(update on sms - R, chain on R).  The
    chain is ~26 m nb^2 flops of GEMMs per panel pair plus a latency floor; the
    update 2 m_k w rest flops (rate = flops per ms on all SMs).  Early steps keep
    r_min (the chain hides under a long update); late steps, where every rank
    waits for the owner's block, give the chain more."""
    upd = 2.0 * mk * w * rest / rate                 # ms on all SMs
    gemm = 26.0 * m_next * nb * nb / rate
    best_r, best_t = r_min, float("inf")
    for r in sorted({r_min, 32, 48, 64, 96}):
        if r < r_min or r >= sms:
            continue
        t = max(upd * sms / (sms - r), lat_ms + gemm * sms / r)
        if t < best_t - 1e-9:
            best_r, best_t = r, t
    return best_r


class CudaOps:
    """Local arithmetic through the C ABI (stream-ordered qrb_op_* calls on
    torch CUDA tensors holding column-major matrices as (cols, ld) tensors)."""

    def __init__(self, world: int = 1, side_lookahead: bool = True):
        import torch
        from . import _native
        self.world = world
        self.lib = _native.load()
        self.native = _native
        # with several ranks a receiver's NCCL kernel can hold SMs while the
        # trailing update starts: let the persistent GEMM hand out tiles dynamically
        _native.set_tuning("nn_dynamic", 1 if world > 1 else 0)
        # the owner's next block is factored on a high-priority side stream
        self.side_lookahead = bool(side_lookahead) and _native.get_tuning("lookahead") > 0
        self.side = torch.cuda.Stream(priority=-1) if self.side_lookahead else None

    @staticmethod
    def _stream():
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def panel_block(self, a, lda, row0, col0, m, w, nb, tau, t2, ldt2, side=False):
        """Block of w <= 2 nb columns at (row0, col0): V in place, tau, merged T2."""
        import torch
        tmp = torch.empty(2 * nb * nb, dtype=torch.float64, device=a.device)
        st = self.lib.qrb_op_panel_block(self._p(a, row0 + col0 * lda), lda, m, w, nb, self._p(tau),
                                         self._p(tmp), self._p(t2), ldt2, self._stream(),
                                         1 if side else 0)
        self.native.check(st, "qrb_op_panel_block")

    def _cap_cols(self, mk, w, m_next, nb, rest):
        """Columns of the owner's update run on the capped grid while the next
        block is factored (the model of qrb_api.cu right_looking)."""
        g = self.native.get_tuning
        sms, r = g("sm_count"), g("la_sms")
        r = min(r, sms // 2)
        rate = 34.0e9  # flop per ms of the DMMA update on all SMs
        tp = g("la_lat_us") * 1e-3 + 26.0 * m_next * nb * nb / (rate * r / sms)
        want = (1.0 + g("la_margin_pct") / 100.0) * tp * rate * (sms - r) / sms / (2.0 * mk * w)
        return min(rest, (int(want) + 63) // 64 * 64), sms - r

    def apply_split(self, v, ldv, m, w, t, ldt, c, ldc, c_off, nc, first, side_work, m_next, nb):
        """C <- Q^T C on nc columns; after the first `first` columns, side_work()
        (the next block's factorization + broadcast) runs on the side stream
        while the rest of the update runs on capped grids.  Returns side_work()."""
        import torch
        main = torch.cuda.current_stream()
        pv, pt, pc = self._p(v), self._p(t), self._p(c, c_off)
        first = min(first, max(nc, 0))
        if nc > 0:
            self.native.check(self.lib.qrb_op_apply_qt_begin(pv, ldv, m, w, pt, ldt, pc, ldc, nc,
                                                             self._stream()), "apply_qt_begin")
            self.native.check(self.lib.qrb_op_apply_qt_cols(pv, ldv, m, w, pc, ldc, 0, first,
                                                            self._stream()), "apply_qt_cols")
        ev = torch.cuda.Event()
        ev.record(main)
        rest = max(nc - first, 0)
        ncap, cap = self._cap_cols(m, w, m_next, nb, rest)
        if self.world > 1:
            # keep SMs free for the whole owner step: the broadcast's NCCL kernel is
            # launched after the side-stream panel and must not wait for a
            # persistent full-grid update to drain (the other ranks wait for it).
            # How many: the split minimising the owner's step (its capped update
            # vs the block chain on the freed SMs) -- late steps, where the chain
            # is the critical path of every rank, give the chain more SMs
            g = self.native.get_tuning
            # (at least 24: the single-GPU default la_sms is 8, but here the
            # broadcast's NCCL CTAs share the freed SMs with the chain)
            cap = g("sm_count") - owner_chain_sms(m, rest, w, m_next, nb, g("sm_count"),
                                                  max(24, g("la_sms")), g("la_lat_us") * 1e-3)
            ncap = rest
        if ncap:
            self.native.set_tuning("grid_cap", cap)
            try:
                self.native.check(self.lib.qrb_op_apply_qt_cols(pv, ldv, m, w, pc, ldc, first, ncap,
                                                                self._stream()), "apply_qt_cols")
            finally:
                self.native.set_tuning("grid_cap", 0)
        if rest - ncap > 0:
            self.native.check(self.lib.qrb_op_apply_qt_cols(pv, ldv, m, w, pc, ldc, first + ncap,
                                                            rest - ncap, self._stream()),
                              "apply_qt_cols")
        # the side work is enqueued after the main stream's update: its host-side
        # CholeskyQR2 flag check then blocks this thread with the GPU already busy
        self.side.wait_event(ev)
        with torch.cuda.stream(self.side):
            res = side_work()
            done = torch.cuda.Event()
            done.record(self.side)
        main.wait_event(done)
        return res

    @staticmethod
    def _p(t, off=0):
        return ctypes.c_void_p(t.data_ptr() + 8 * off)

    def panel(self, a, lda, row0, col0, m, w, tau, t, ldt):
        st = self.lib.qrb_op_panel(self._p(a, row0 + col0 * lda), lda, m, w, self._p(tau),
                                   self._p(t), ldt, None)
        self.native.check(st, "qrb_op_panel")

    def apply_qt(self, v, ldv, v_off, m, w, t, ldt, c, ldc, c_off, nc):
        if nc <= 0:
            return
        st = self.lib.qrb_op_apply_qt(self._p(v, v_off), ldv, m, w, self._p(t), ldt,
                                      self._p(c, c_off), ldc, nc, None)
        self.native.check(st, "qrb_op_apply_qt")

    def trsm_upper(self, r, ldr, r_off, n, b, ldb, b_off, nrhs):
        """b[b_off : b_off+n] <- R^-1 b for the n x n upper block starting at element r_off."""
        st = self.lib.qrb_op_trsm_upper(self._p(r, r_off), ldr, n, 16,
                                        self._p(b, b_off), ldb, nrhs, None)
        self.native.check(st, "qrb_op_trsm_upper")

    def gemm_nn_sub(self, a, lda, a_off, m, k, bmat, ldb, b_off, c, c_off, n):
        """c[c_off : c_off+m] -= A (m x k at a + a_off) @ bmat[b_off : b_off+k]."""
        st = self.lib.qrb_op_gemm_nn_sub(self._p(a, a_off), lda, self._p(bmat, b_off), ldb,
                                         self._p(c, c_off), ldb, m, n, k, None)
        self.native.check(st, "qrb_op_gemm_nn_sub")

    def sync(self):
        import torch
        torch.cuda.synchronize()


@dataclass
class DistFactors:
    m: int
    n: int
    nb: int
    lda: int
    rank: int
    world: int
    a_local: object                     # torch (n_local, lda): factored local panels
    t_all: object                       # torch (npanels*nb, nb): T_k of every panel (rows = T columns)
    tau_all: object = None
    factor_seconds: float = 0.0
    stats: dict = field(default_factory=dict)
    bw: int = 0                         # column block width of the layout (0 = nb)
    t2_blocks: object = None            # torch (nblocks, 2nb, 2nb): merged reflector of every
                                        #   panel-pair block, column-major (bw = 2 nb only)

    @property
    def block(self) -> int:
        return self.bw or self.nb


def _panel_views(buf, m: int, n: int, nb: int, k: int):
    j0 = k * nb
    pw = min(nb, n - j0)
    mk = m - j0
    ldv = mk + (mk & 1)
    nelem = ldv * pw + nb * nb + nb
    return (j0, pw, mk, ldv, nelem, buf[: ldv * pw].view(pw, ldv),
            buf[ldv * pw: ldv * pw + nb * nb].view(nb, nb), buf[ldv * pw + nb * nb: nelem])


def factorize_distributed(a_local, m: int, n: int, nb: int, lda: int, rank: int, world: int,
                          ops, group=None, lookahead: bool = True, bw: int | None = None,
                          host_src=None, chunk_cols: int = 2048) -> DistFactors:
    """Blocked Householder QR of the block-cyclic matrix (blocks of bw = nb or
    2 nb columns); a_local is overwritten with the local blocks of the factored
    matrix (R above, V below).

    With ``lookahead`` (depth 1) the owner of block k+1 first applies Q_k^T to
    that block only, factors it and starts its broadcast, and only then updates
    the rest of its trailing columns; the other ranks receive block k+1 while
    they are still busy with step k.  Each rank factors 1/G of the blocks, so
    the panel latency is spread over the G GPUs instead of serialising every
    step.  If ``ops.side_lookahead`` the owner's factorization and broadcast
    run on a second stream concurrently with its own update (ops.apply_split).
    Blocks travel in two alternating buffers.

    ``host_src`` (pinned host tensor shaped like a_local): the local blocks are
    copied in by column chunks on a copy stream inside the timed region, and
    until the last chunk has landed every step updates its columns chunk by
    chunk, each after its chunk's copy event -- the host-to-device transfer
    overlaps the first steps (the end-to-end path of bench.py).
    """
    import torch
    import torch.distributed as dist

    bw = bw or nb
    if bw % nb or bw > 2 * nb:
        raise ValueError("block width must be nb or 2 nb")
    nblk = -(-n // bw)
    npan = -(-n // nb)
    dev = a_local.device
    dt = torch.float64
    t_all = torch.zeros((npan * nb, nb), dtype=dt, device=dev)
    tau_all = torch.zeros(npan * nb, dtype=dt, device=dev)
    ldv_max = m + (m & 1)
    bufs = [torch.empty(ldv_max * bw + bw * bw + bw, dtype=dt, device=dev) for _ in range(2)]
    n_local = a_local.shape[0]
    side = bool(getattr(ops, "side_lookahead", False))
    stats = {"bytes_broadcast": 0, "panels": npan, "blocks": nblk, "block_width": bw,
             "lookahead": bool(lookahead and world > 1), "side_lookahead": side}

    def views(k):
        buf = bufs[k % 2]
        j0 = k * bw
        w = min(bw, n - j0)
        mk = m - j0
        ldv = mk + (mk & 1)
        nelem = ldv * w + bw * bw + bw
        return (j0, w, mk, ldv, nelem, buf[: ldv * w].view(w, ldv),
                buf[ldv * w: ldv * w + bw * bw].view(bw, bw), buf[ldv * w + bw * bw: nelem])

    def factor_and_pack(k, on_side=False):
        j0, w, mk, ldv, nelem, vview, t2view, tauv = views(k)
        lcol = (k // world) * bw
        t2view.zero_()
        ops.panel_block(a_local, lda, j0, lcol, mk, w, nb, tauv, t2view, bw, side=on_side)
        vview[:, :mk].copy_(a_local[lcol:lcol + w, j0:m])

    def start_bcast(k):
        nelem = views(k)[4]
        if world == 1:
            return None
        stats["bytes_broadcast"] += 8 * nelem
        return dist.broadcast(bufs[k % 2][:nelem], src=owner_of(k, world), group=group,
                              async_op=True)

    t2_blocks = (torch.zeros((nblk, bw, bw), dtype=dt, device=dev) if bw == 2 * nb else None)

    def unpack(k):  # per-panel T factors (diagonal blocks of T2), the block's T2, tau
        j0, w, mk, ldv, nelem, vview, t2view, tauv = views(k)
        if t2_blocks is not None:
            t2_blocks[k].copy_(t2view)
        for p in range(-(-w // nb)):
            pw = min(nb, w - p * nb)
            kp = j0 // nb + p
            t_all[kp * nb:kp * nb + pw, :pw].copy_(t2view[p * nb:p * nb + pw, p * nb:p * nb + pw])
        tau_all[j0:j0 + w].copy_(tauv[:w])

    def apply(k, col_from, col_to):
        if col_to <= col_from:
            return
        j0, w, mk, ldv, _, vview, t2view, _ = views(k)
        ops.apply_qt(vview, ldv, 0, mk, w, t2view, bw, a_local, lda, j0 + col_from * lda,
                     col_to - col_from)

    la = lookahead and world > 1
    ops.sync()
    t0 = time.perf_counter()
    ev = None
    if a_local.is_cuda:                  # device time of the whole factorization
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    # chunked host -> device copy of the local blocks (overlapped with the first steps)
    chunks, landed, waited = [], [], [0]
    if host_src is not None:
        cstream = torch.cuda.Stream()
        cstream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cstream):
            for c0 in range(0, n_local, chunk_cols):
                c1 = min(n_local, c0 + chunk_cols)
                a_local[c0:c1].copy_(host_src[c0:c1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(cstream)
                chunks.append((c0, c1))
                landed.append(e)
        stats["h2d_chunks"] = len(chunks)

    def all_landed():
        return not landed or waited[0] == len(landed) or landed[-1].query()

    def need(col_to):
        """the current stream waits for the copies of local columns [0, col_to)"""
        while waited[0] < len(landed) and chunks[waited[0]][0] < col_to:
            torch.cuda.current_stream().wait_event(landed[waited[0]])
            waited[0] += 1

    def apply_chunked(k, col_from, col_to):
        for c0, c1 in chunks:
            lo, hi = max(c0, col_from), min(c1, col_to)
            if lo < hi:
                need(hi)
                apply(k, lo, hi)

    if rank == owner_of(0, world):
        need(bw)
        factor_and_pack(0)
    pending = start_bcast(0)
    for k in range(nblk):
        if not all_landed():
            # copies still in flight: the serial schedule, column chunk by chunk
            if pending is not None:
                pending.wait()
            unpack(k)
            lfirst = first_local_after(k, rank, world) * bw
            nxt = k + 1
            pending = None
            if nxt < nblk and rank == owner_of(nxt, world):
                w1 = min(bw, n - nxt * bw)
                apply_chunked(k, lfirst, lfirst + w1)
                factor_and_pack(nxt)
                pending = start_bcast(nxt)
                apply_chunked(k, lfirst + w1, n_local)
            else:
                if nxt < nblk:
                    pending = start_bcast(nxt)
                apply_chunked(k, lfirst, n_local)
            continue
        need(n_local)
        if pending is not None:
            pending.wait()
        unpack(k)
        lfirst = first_local_after(k, rank, world) * bw
        nxt = k + 1
        pending = None
        if nxt < nblk and rank == owner_of(nxt, world):
            # block k+1 is this rank's local block starting at lfirst
            w1 = min(bw, n - nxt * bw)
            if side:
                j0, w, mk, ldv, _, vview, t2view, _ = views(k)

                def side_work(nxt=nxt):
                    factor_and_pack(nxt, on_side=True)
                    return start_bcast(nxt)
                pending = ops.apply_split(vview, ldv, mk, w, t2view, bw, a_local, lda,
                                          j0 + lfirst * lda, n_local - lfirst, w1, side_work,
                                          m - nxt * bw, nb)
                continue
            apply(k, lfirst, lfirst + w1)
            factor_and_pack(nxt)
            if la:
                pending = start_bcast(nxt)
            apply(k, lfirst + w1, n_local)
            if not la:
                pending = start_bcast(nxt)
        else:
            if la and nxt < nblk:
                pending = start_bcast(nxt)   # receive while updating
            apply(k, lfirst, n_local)
            if not la and nxt < nblk:
                pending = start_bcast(nxt)
    if ev is not None:
        ev[1].record()
    ops.sync()
    secs = time.perf_counter() - t0
    if ev is not None:
        stats["wall_seconds"] = secs
        secs = ev[0].elapsed_time(ev[1]) / 1e3
    return DistFactors(m, n, nb, lda, rank, world, a_local, t_all, tau_all, secs, stats, bw,
                       t2_blocks)


def gather_factored(f: DistFactors, group=None, place=None):
    """All ranks receive every factored panel.  With ``place(k, panel)`` each
    (pw, lda) panel view is handed to the caller (e.g. copied straight into a
    QrDevice); otherwise the full (n, lda) tensor is returned."""
    import torch
    import torch.distributed as dist

    npan = -(-f.n // f.nb)
    max_local = max(local_cols(f.n, f.block, r, f.world) for r in range(f.world))
    dev = f.a_local.device
    send = torch.zeros((max_local, f.lda), dtype=torch.float64, device=dev)
    send[: f.a_local.shape[0]].copy_(f.a_local)
    if f.world > 1:
        recv = torch.empty((f.world * max_local, f.lda), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(recv, send, group=group)
    else:
        recv = send
    full = None if place else torch.empty((f.n, f.lda), dtype=torch.float64, device=dev)
    for k in range(npan):
        r, lc = panel_home(k, f.nb, f.block, f.world)
        pw = min(f.nb, f.n - k * f.nb)
        src = recv[r * max_local + lc: r * max_local + lc + pw]
        if place:
            place(k, src)
        else:
            full[k * f.nb:k * f.nb + pw].copy_(src)
    return full


def gather_storage(n: int, bw: int, world: int, lda: int, device):
    """Device storage for gather_into: (rounds * world * bw, lda) columns."""
    import torch
    rounds = -(-(-(-n // bw)) // world)
    return torch.empty((rounds * world * bw, lda), dtype=torch.float64, device=device)


def gather_into(f: DistFactors, out, group=None):
    """Every rank receives the whole factored matrix straight into ``out``
    (gather_storage) in global column order: round i all-gathers every
    rank's i-th local block, and the blocks of round i are the consecutive
    global blocks i*world .. i*world + world - 1 -- no receive buffer and no
    reordering copy (gather_factored needs both).  A QrDevice.view over out[:n]
    then solves without a library-owned copy of the factors."""
    import torch
    import torch.distributed as dist

    bw = f.block
    nblk = -(-f.n // bw)
    rounds = -(-nblk // f.world)
    send = torch.zeros((bw, f.lda), dtype=torch.float64, device=f.a_local.device)
    n_local = f.a_local.shape[0]
    for i in range(rounds):
        dst = out[i * f.world * bw:(i + 1) * f.world * bw]
        c0 = i * bw
        w = max(0, min(bw, n_local - c0))
        if f.world == 1:
            dst[:w].copy_(f.a_local[c0:c0 + w])
            continue
        if w == bw:
            src = f.a_local[c0:c0 + bw]
        else:                            # a short last block, or none: zero padded
            send.zero_()
            if w:
                send[:w].copy_(f.a_local[c0:c0 + w])
            src = send
        dist.all_gather_into_tensor(dst, src, group=group)
    return out


def singular_column(diag: np.ndarray, block: int) -> int:
    """First bad pivot in the reference's bottom-up tile order, or -1
    (kernels.py:423-426 inside tiles visited from the last, task_engine.py:246-253)."""
    n = diag.size
    block = block if block > 0 else max(n, 1)
    for t in range(-(-n // block) - 1, -1, -1):
        seg = diag[t * block:min(n, (t + 1) * block)]
        bad = np.flatnonzero(~(np.abs(seg) >= 1e-300))
        if bad.size:
            return t * block + int(bad[0])
    return -1


def global_rdiag(f: DistFactors, group=None) -> np.ndarray:
    """diag(R) (n values, host) from every rank's factored blocks (one all-reduce)."""
    import torch
    import torch.distributed as dist
    d = torch.zeros(f.n, dtype=torch.float64, device=f.a_local.device)
    bw = f.block
    for i, k in enumerate(local_panels(-(-f.n // bw), f.rank, f.world)):
        c0, w = k * bw, min(bw, f.n - k * bw)
        cols = torch.arange(w, device=d.device)
        d[c0:c0 + w] = f.a_local[i * bw + cols, c0 + cols]
    if f.world > 1:
        dist.all_reduce(d, group=group)
    return d.cpu().numpy()


def check_singular(f: DistFactors, report_block: int | None = None, group=None) -> None:
    """Raise SingularMatrixError on EVERY rank with the column the reference's
    solve would report (tiles of report_block visited bottom-up)."""
    bad = singular_column(global_rdiag(f, group), report_block or f.n)
    if bad >= 0:
        raise SingularMatrixError(bad)


def solve_distributed(f: DistFactors, b_share, ops, group=None, report_block: int | None = None):
    """Memory-lean multi-GPU solve (no factor replication; config 4 at 8 GPUs):
    every rank keeps only its own panels and solves its slice share b_share
    (torch (s, lda), s may be 0).

    Q^T B: panel by panel the owner broadcasts the packed reflector block
    (same buffer as the factorization) and every rank applies it to its
    slices.  R^-1: block column by block column from the bottom, the owner
    broadcasts R[0:i1, block k]; every rank solves its diagonal block and
    updates the rows above.  Traffic = one pass over V and R per solve, no
    all-gather of the factored matrix.  Returns (x (s, n), resid (s,)).
    """
    import torch
    import torch.distributed as dist

    m, n, nb, lda, rank, world = f.m, f.n, f.nb, f.lda, f.rank, f.world
    check_singular(f, report_block, group)          # before any work (reference order)
    npan = -(-n // nb)
    dev = f.a_local.device
    s = b_share.shape[0]
    y = b_share.clone()
    buf = torch.empty((m + (m & 1)) * nb + nb * nb + nb, dtype=torch.float64, device=dev)
    for k in range(npan):
        j0, pw, mk, ldv, nelem, vview, tview, _ = _panel_views(buf, m, n, nb, k)
        own, lcol = panel_home(k, nb, f.block, world)
        if rank == own:
            vview[:, :mk].copy_(f.a_local[lcol:lcol + pw, j0:m])
            tview.copy_(f.t_all[k * nb:(k + 1) * nb])
        if world > 1:
            dist.broadcast(buf[:nelem], src=own, group=group)
        if s:
            ops.apply_qt(vview, ldv, 0, mk, pw, tview, nb, y, lda, j0, s)
    resid = torch.linalg.norm(y[:, n:m], dim=1) if s else torch.zeros(0, device=dev)
    rflat = torch.empty(nb * (n + 2), dtype=torch.float64, device=dev)
    for k in range(npan - 1, -1, -1):
        i0 = k * nb
        bs = min(nb, n - i0)
        i1 = i0 + bs
        ldr = i1 + (i1 & 1)
        rblk = rflat[: bs * ldr].view(bs, ldr)      # R[0:i1, block k], column-major, ld = ldr
        own, lcol = panel_home(k, nb, f.block, world)
        if rank == own:
            rblk[:, :i1].copy_(f.a_local[lcol:lcol + bs, :i1])
        if world > 1:
            dist.broadcast(rblk, src=own, group=group)
        if s:
            ops.trsm_upper(rblk, ldr, i0, bs, y, lda, i0, s)
            if i0 > 0:
                ops.gemm_nn_sub(rblk, ldr, 0, i0, bs, y, lda, i0, y, 0, s)
    ops.sync()
    return y[:, :n], resid


def memory_plan(m: int, n: int, nb: int, world: int, hbm_bytes: float, bw: int | None = None,
                headroom: float = 0.8) -> dict:
    """Per-rank HBM plan of the multi-GPU factorization + solve (bytes).

    local: this layout's largest local share of A (column blocks of bw = 2 nb,
    block k on rank k % world); bcast: the two alternating (V, T2, tau) block
    buffers of factorize_distributed; t_tau: T of every panel + tau; replica:
    what the replicated solve adds (a full QrDevice copy of the factors plus
    gather_factored's all-gather receive buffer).  The solve replicates only if
    local + bcast + t_tau + replica fits ``headroom`` of the HBM, otherwise it is
    the memory-lean streamed solve (solve_distributed).
    """
    bw = bw or 2 * nb
    lda = (m + 31) // 32 * 32
    max_local = max(local_cols(n, bw, r, world) for r in range(world))
    local = 8.0 * lda * max_local
    bcast_each = 8.0 * ((m + (m & 1)) * bw + bw * bw + bw)
    npan = -(-n // nb)
    t_tau = 8.0 * (npan * nb * nb + npan * nb)
    replica = 8.0 * lda * n + 8.0 * world * max_local * lda
    base = local + 2 * bcast_each + t_tau
    lean = base + replica > headroom * hbm_bytes
    return {"lda": lda, "block_width": bw, "local_cols": max_local, "local_bytes": local,
            "bcast_buffer_bytes": bcast_each, "bcast_buffers": 2, "t_tau_bytes": t_tau,
            "replica_bytes": replica, "total_bytes": base + (0.0 if lean else replica),
            "lean_solve": lean, "fits": base <= headroom * hbm_bytes}


def scatter_block_cyclic(a_full_cols, n: int, nb: int, rank: int, world: int):
    """This rank's local panels (torch (n_local, lda)) from a full (n, lda) tensor."""
    import torch
    npan = -(-n // nb)
    parts = [a_full_cols[k * nb:min(n, (k + 1) * nb)] for k in local_panels(npan, rank, world)]
    if not parts:
        return a_full_cols[:0].clone()
    return torch.cat(parts, dim=0).contiguous()


def slice_share(s: int, rank: int, world: int) -> tuple[int, int]:
    """[first, count) of the slices this rank solves."""
    base, rem = divmod(s, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


# -- benchmark rank (bench.py under torchrun) -----------------------------------------------


def bench_rank(args, rank: int, world: int):
    import json
    import os

    import torch
    import torch.distributed as dist

    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    backend = getattr(args, "dist_backend", "nccl")
    # NCCL kernels hold one SM per channel while they wait for the owner's block;
    # a receiver posts its broadcast before its update, so cap the CTAs a
    # collective may take (the 70 MB block still moves in < 1 ms over NVLink)
    os.environ.setdefault("NCCL_MAX_CTAS", "8")
    if backend == "gloo":
        # functional check of this multi-rank bench path on a one-GPU box: the
        # ranks share the GPU and exchange through host memory (no performance
        # meaning; the driver's multi-GPU runs use NCCL, one GPU per rank)
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    if backend == "gloo":
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local_rank))
    from bench import (CUBLAS_DGEMM_TFLOPS, FP64_NOMINAL_TFLOPS, FP64_PEAK_TFLOPS, METRIC, UNIT,
                       ClockSampler, build_workload, emit, qr_flops, solve_flops)
    from . import ct_system as cs
    from .device import QrDevice, launch_count

    g, _, x_true, S = build_workload(args.config, args.slices, host_coo=False)
    m, n, nb = g.n_rays, g.n_pixels, args.nb
    bw = 2 * nb  # panel pairs: K = 2nb trailing-update GEMMs, one broadcast per pair
    lda = (m + 31) // 32 * 32
    # each rank densifies only its own block-cyclic column blocks on its GPU
    a_pristine = cs.densify_device(g, lda, rank=rank, world=world, nb=bw)
    cols = [c for k in local_panels(-(-n // bw), rank, world)
            for c in range(k * bw, min(n, (k + 1) * bw))]
    xt = torch.from_numpy(np.ascontiguousarray(x_true[cols].T)).cuda()
    ax = xt @ a_pristine[:, :m]                       # this rank's share of A x
    if world > 1:
        dist.all_reduce(ax)
    b_host = cs.noisy_sinograms(ax.cpu().numpy().T, args.config)
    del xt, ax
    torch.cuda.empty_cache()
    first, cnt = slice_share(S, rank, world)
    b_dev = torch.zeros((max(cnt, 1), lda), dtype=torch.float64, device="cuda")
    b_dev[:cnt, :m] = torch.from_numpy(np.ascontiguousarray(b_host[:, first:first + cnt].T)).cuda()
    x_dev = torch.zeros((max(cnt, 1), n + (n & 1)), dtype=torch.float64, device="cuda")
    ops = CudaOps(world)
    # keep a pristine copy of the local panels only if it fits (config 4 at 8 GPUs
    # is ~71 GB per rank: re-densify with the Siddon kernel instead)
    free, total = torch.cuda.mem_get_info()
    if 8 * a_pristine.numel() < 0.4 * free:
        a_local = torch.empty_like(a_pristine)
        reset = lambda: a_local.copy_(a_pristine)  # noqa: E731
    else:
        a_local, a_pristine = a_pristine, None

        def reset():
            a_local.zero_()
            cs.densify_into(g, a_local, lda, rank=rank, world=world, nb=bw)
    # replicate the factors for the solve only if a full copy (plus the gather
    # buffer) fits next to the local panels; otherwise stream V and R (config 4)
    free, total = torch.cuda.mem_get_info()
    plan = memory_plan(m, n, nb, world, free + 8.0 * a_local.numel(), bw=bw)
    lean = args.lean_solve or plan["lean_solve"]
    # replicated solve: the factors are all-gathered straight into one buffer in
    # global column order and solved through a handle over it (no second copy)
    gstore = None if lean else gather_storage(n, bw, world, lda, a_local.device)
    q = None if lean else QrDevice.view(gstore, m, n, nb, local_rank)

    def step():
        reset()
        f = factorize_distributed(a_local, m, n, nb, lda, rank, world, ops, bw=bw)
        t1 = time.perf_counter()
        if lean:
            torch.cuda.synchronize()
            ts = time.perf_counter()
            solve_distributed(f, b_dev[:cnt], ops)
            return f.factor_seconds, 0.0, time.perf_counter() - ts
        gather_into(f, gstore)
        q.set_factors(f.tau_all.cpu().numpy()[:n], f.t_all.cpu().numpy().T.copy(order="F"))
        if f.t2_blocks is not None:
            q.set_pair_factors(f.t2_blocks)
        t2 = time.perf_counter()
        srep = q.solve_device(b_dev[:cnt], x_dev[:cnt]) if cnt else {"total_ms": 0.0}
        return f.factor_seconds, t2 - t1, srep["total_ms"] / 1e3

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        sampler.start()
    l0 = launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fs, gs, ss = [], [], []
    for _ in range(args.steps):
        a, b, c = step()
        fs.append(a)
        gs.append(b)
        ss.append(c)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    step_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    f_s = torch.tensor([float(np.mean(fs))], device="cuda")
    s_s = torch.tensor([float(np.mean(ss))], device="cuda")
    # the replicated solve pays for the factor all-gather once per factorization:
    # slices/s is reported with it included (solve-only beside it)
    sg_s = torch.tensor([float(np.mean(ss)) + float(np.mean(gs))], device="cuda")
    for t in (step_ms, f_s, s_s, sg_s):
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    clocks = sampler.stop() if sampler else None
    launches = launch_count() - l0

    # config 5: a 4096-slice batch on the config-3 factors, slices split over the
    # ranks (no communication in the solve); sinograms from the all-reduced
    # per-rank products A_local x_local
    cfg5 = None
    if args.config == 3 and getattr(args, "cfg5_slices", 0) > 0 and not lean:
        S5 = args.cfg5_slices
        x5 = cs.phantom_stack_device(5, S5)                        # (S5, n)
        ax5 = x5[:, cols] @ a_pristine[:, :m] if a_pristine is not None else None
        if ax5 is None:                                            # no pristine copy kept
            reset()
            ax5 = x5[:, cols] @ a_local[:, :m]
        del x5
        if world > 1:
            dist.all_reduce(ax5)
        f5, c5 = slice_share(S5, rank, world)
        b5h = cs.noisy_sinograms(ax5.cpu().numpy().T, 5)           # (m, S5), same seeds as N = 1
        del ax5
        b5 = torch.zeros((max(c5, 1), lda), dtype=torch.float64, device="cuda")
        b5[:c5, :m] = torch.from_numpy(np.ascontiguousarray(b5h[:, f5:f5 + c5].T)).cuda()
        del b5h
        x5o = torch.zeros((max(c5, 1), n + (n & 1)), dtype=torch.float64, device="cuda")
        if c5:
            q.solve_device(b5[:c5], x5o[:c5])                       # warm-up
        dist.barrier()
        t5 = []
        for _ in range(2):
            ms = q.solve_device(b5[:c5], x5o[:c5])["total_ms"] if c5 else 0.0
            t5.append(ms)
        s5 = torch.tensor([float(np.mean(t5))], device="cuda")
        dist.all_reduce(s5, op=dist.ReduceOp.MAX)
        cfg5 = {"workload": f"config5: solve {S5} slices on the config-3 factors, "
                            f"{S5 // world}+ per GPU", "slices": S5, "solve_ms": float(s5),
                "slices_per_s": S5 / (float(s5) * 1e-3),
                "solve_tflops": solve_flops(m, n, S5) / (float(s5) * 1e-3) / 1e12}
        del b5, x5o
        torch.cuda.empty_cache()

    # end to end through host buffers: this rank's panels from pinned host memory
    # in, its slice share of X out (factorization + gather + solve inside)
    reset()
    from .device import PinnedHostArray
    a_pin_hold = PinnedHostArray(tuple(a_local.shape))      # exact size (no power-of-2 rounding)
    a_pin = torch.from_numpy(a_pin_hold.array)
    a_pin.copy_(a_local)
    b_pin = torch.empty((max(cnt, 1), lda), dtype=torch.float64, pin_memory=True)
    b_pin.copy_(b_dev)
    x_pin = torch.empty((max(cnt, 1), n), dtype=torch.float64, pin_memory=True)
    dist.barrier()
    torch.cuda.synchronize()
    t_e2e = time.perf_counter()
    f = factorize_distributed(a_local, m, n, nb, lda, rank, world, ops, bw=bw, host_src=a_pin)
    if lean:
        b_dev[:cnt].copy_(b_pin[:cnt], non_blocking=True)
        xs, _ = solve_distributed(f, b_dev[:cnt], ops)
        x_pin[:cnt].copy_(xs)
    else:
        gather_into(f, gstore)
        q.set_factors(f.tau_all.cpu().numpy()[:n], f.t_all.cpu().numpy().T.copy(order="F"))
        if f.t2_blocks is not None:
            q.set_pair_factors(f.t2_blocks)
        if cnt:
            q.solve(b_pin.numpy().T[:m, :cnt], out=x_pin.numpy().T[:, :cnt])
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t_e2e], device="cuda")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    if rank == 0:
        fl = qr_flops(m, n)
        value = fl / float(f_s) / 1e12
        n_dev = min(world, torch.cuda.device_count())
        if backend == "gloo":
            # functional mode: the ranks share the box's GPU(s) and exchange
            # through host memory -- not a multi-GPU measurement
            parallelism = (f"FUNCTIONAL CHECK, not a multi-GPU measurement: {world} ranks sharing "
                           f"{n_dev} GPU(s), gloo (host-mediated) block broadcast, 1D block-cyclic "
                           f"column blocks of {bw}; slices split for the solve")
        else:
            parallelism = (f"1D block-cyclic column blocks of {bw} (panel pairs, nb={nb}) over "
                           f"{world} GPUs, NCCL block broadcast, owner look-ahead on a side "
                           f"stream; slices split for the solve")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_dev, "ranks": world,
            "backend": backend, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(step_ms), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Siddon fan-beam A, seeded phantoms, 1% noise)",
            "config": {"workload": f"config{args.config}: QR of A {m}x{n} + solve {S} slices",
                       "m": m, "n": n, "slices": S, "panel_width": nb,
                       "parallelism": parallelism,
                       "l2": "inputs (A = %.1f GB) larger than L2 (126 MB)" % (m * n * 8 / 1e9)},
            "pct_fp64_peak": value / (FP64_PEAK_TFLOPS * n_dev),
            "pct_fp64_nominal": value / (FP64_NOMINAL_TFLOPS * n_dev),
            "vs_cublas_dgemm": value / (CUBLAS_DGEMM_TFLOPS * n_dev),
            "slices_per_s": S / float(sg_s),
            "slices_per_s_solve_only": S / float(s_s),
            "solve_tflops": solve_flops(m, n, S) / float(s_s) / 1e12,
            "factor_ms": float(f_s) * 1e3, "gather_ms": float(np.mean(gs)) * 1e3,
            "solve_path": "streamed V/R broadcast (no replication)" if lean else
                          "all-gathered factors, per-rank solve",
            "gpu_launches": int(launches), "clocks": clocks,
            "roofline": {"bound": "tensor", "achieved": value / n_dev,
                         "peak": FP64_PEAK_TFLOPS, "unit": UNIT,
                         "frac": value / n_dev / FP64_PEAK_TFLOPS, "traffic": None,
                         "kernel": "whole factorization per GPU (CUDA events, max over "
                                   "ranks); per-kernel accounting is single-GPU only"},
            "config5": cfg5,
            "e2e": {"value": fl / float(e2e_s) / 1e12, "unit": UNIT,
                    "h2d_bytes_per_step": int(8 * lda * n + 8 * m * S),
                    "d2h_bytes_per_step": int(8 * n * S),
                    "ms_per_step": float(e2e_s) * 1e3,
                    "path": "pinned host blocks (chunked H2D overlapped with the first steps) -> "
                            "factorize_distributed -> " +
                            ("streamed V/R solve" if lean else "all-gather -> QrDevice.solve") +
                            " (host B share -> host X share); max over ranks"},
        }
        emit(line)
    dist.destroy_process_group()
