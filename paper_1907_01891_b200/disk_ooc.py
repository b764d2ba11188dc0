"""Disk-staged QR and solve: matrices larger than host memory (the paper's SSD regime).

The reference is an out-of-core engine first: tiles live on disk, a bounded
RAM cache and ONE prefetch / write-back agent keep the compute fed, and the
task order is left-looking so every produced tile is written once
(task_engine.py:4-9, 187-217, 330-474; tile_store.py:225-415).
:mod:`ooc` covers "larger than HBM, fits in host RAM" by pinning the whole
matrix; this module covers "larger than host RAM": nothing but a few pinned
panel buffers is ever resident on the host.

Left-looking by super-panels sized to the HBM budget:

  for each super-panel S (as many nb-wide panels as fit in HBM):
      disk -> pinned -> HBM   the columns of S from the input store
      for every earlier panel k: disk -> pinned -> HBM the reflectors V_k
          (rows >= k*nb of the factored store), apply Q_k^T to S
      factor S in HBM (panel kernels + DMMA trailing updates)
      HBM -> pinned -> disk   S into the factored store (written once)

I/O is panel-granular: tiles are column-major on disk, so the nb columns of a
panel inside one tile are ONE contiguous positional read / write
(TiledMatrix.read_columns / write_columns).  A small thread pool (the
reference's I/O agent, task_engine.py:330-474) reads panel k+1 and k+2 into
pinned buffers while the GPU applies panel k; the H2D copies run on their own
stream, ordered with the compute stream by CUDA events; write-back of a
finished super-panel overlaps the next super-panel's reads.  T factors and tau
(small) stay in HBM.  The solve streams V once for Q^T B and R once for the
back substitution.
"""

from __future__ import annotations

import ctypes
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _native
from .errors import SingularMatrixError
from .ooc import _StagedFactors
from .tile_store import TiledMatrix


def _p(t, off: int = 0) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() + 8 * off)


class DiskStagedQR(_StagedFactors):
    """QR of the tiled matrix ``src`` (m x n on disk) into the tiled store
    ``dst`` (R on/above the diagonal, unit-lower reflectors below, the
    reference's factored layout), using at most ``budget_bytes`` of HBM for the
    super-panel.  ``src`` may be None when only solving with existing factors."""

    def __init__(self, src: TiledMatrix | None, dst: TiledMatrix, nb: int = 128,
                 budget_bytes: int = 32 << 30, io_threads: int = 2, page_cache: bool = True):
        """``page_cache=False``: every read comes from the device and every write
        is synced to it and dropped from the OS page cache (TiledMatrix.uncached)
        -- how the engine behaves when the host has no RAM to spare for caching."""
        import torch

        m, n = dst.rows, dst.cols
        if m < n:
            raise ValueError(f"matrix must have rows >= cols, got {m}x{n}")
        if src is not None and (src.rows, src.cols) != (m, n):
            raise ValueError("source and factor stores differ in shape")
        self.lib = _native.load()
        self.src, self.dst = src, dst
        for st in (src, dst):
            if st is not None:
                st.uncached = not page_cache
        self.m, self.n, self.nb = m, n, nb
        self.lda = (m + 31) // 32 * 32
        self.npan = -(-n // nb)
        self.sp_cols = self.super_panel_cols(n, nb, self.lda, budget_bytes)
        dev = torch.device("cuda")
        self._init_factors(dev)
        self.copy_stream = torch.cuda.Stream()
        self.pool = ThreadPoolExecutor(max_workers=max(1, io_threads))     # reads
        self.wpool = ThreadPoolExecutor(max_workers=max(1, io_threads))    # write-back
        self.hbuf = [torch.empty((2 * nb, self.lda), dtype=torch.float64, pin_memory=True)
                     for _ in range(2)]
        # write-back ring: bounded pinned memory, a slot is reused once its write is done
        self.wbuf = [torch.empty((nb, self.lda), dtype=torch.float64, pin_memory=True)
                     for _ in range(3)]
        self.wfut: list = [None] * len(self.wbuf)
        self._wslot = 0
        self.dbuf = [torch.empty((2 * nb, self.lda), dtype=torch.float64, device=dev)
                     for _ in range(2)]
        self.stats: dict = {}
        self._io = {"read_bytes": 0, "write_bytes": 0, "read_s": 0.0, "write_s": 0.0}

    def close(self) -> None:
        self.pool.shutdown(wait=True)
        self.wpool.shutdown(wait=True)

    # -- I/O -------------------------------------------------------------------------
    def _read(self, store: TiledMatrix, k: int, row0: int, row1: int | None, w: int, hb,
              wait_evt):
        """Worker: columns [k nb, k nb + w) rows [row0, row1) of ``store`` into
        the pinned buffer hb."""
        if wait_evt is not None:
            wait_evt.synchronize()          # the previous H2D out of hb has finished
        c0 = k * self.nb
        t0 = time.perf_counter()
        view = hb.numpy().T                 # (lda, nb) Fortran
        store.read_columns(c0, w, row0, view, row1)
        r1 = self.m if row1 is None else row1
        self._io["read_bytes"] += 8 * w * (r1 - row0)
        self._io["read_s"] += time.perf_counter() - t0

    def _stream(self, store: TiledMatrix, items, consume) -> None:
        """Double-buffered disk -> pinned -> HBM pipeline over ``items`` =
        [(k, row0, row1, width)] (columns [k nb, k nb + width)), calling
        consume(item, device_buffer) on the current stream for each, in order."""
        import torch

        cur = torch.cuda.current_stream()
        h2d = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]
        h2d_recorded = [False, False]
        futs = {}

        def submit(idx):
            if idx < len(items):
                s = idx % 2
                k, r0, r1, w = items[idx][:4]
                futs[idx] = self.pool.submit(self._read, store, k, r0, r1, w, self.hbuf[s],
                                             h2d[s] if h2d_recorded[s] else None)

        submit(0)
        submit(1)
        for idx, item in enumerate(items):
            k, r0, r1, w = item[:4]
            s = idx % 2
            futs.pop(idx).result()
            r1 = self.m if r1 is None else r1
            with torch.cuda.stream(self.copy_stream):
                self.copy_stream.wait_event(used[s])
                self.dbuf[s][:w, r0:r1].copy_(self.hbuf[s][:w, r0:r1], non_blocking=True)
                h2d[s].record(self.copy_stream)
                h2d_recorded[s] = True
            submit(idx + 2)                 # waits on h2d[s] before refilling hbuf[s]
            cur.wait_event(h2d[s])
            consume(item, self.dbuf[s])
            used[s].record(cur)

    def _write_superpanel(self, d, c0: int, c1: int) -> list:
        """Queue D2H + positional tile writes of columns [c0, c1) (device block d)
        through the bounded pinned ring."""
        import torch

        futs = []
        nb = self.nb
        for k0 in range(c0, c1, nb):
            w = min(nb, c1 - k0)
            slot = self._wslot
            self._wslot = (slot + 1) % len(self.wbuf)
            if self.wfut[slot] is not None:
                self.wfut[slot].result()    # slot free again
            host = self.wbuf[slot]
            host[:w].copy_(d[k0 - c0:k0 - c0 + w], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()

            def work(host=host, ev=ev, k0=k0, w=w):
                ev.synchronize()
                t0 = time.perf_counter()
                self.dst.write_columns(k0, w, host[:w].numpy().T[:self.m])
                self._io["write_bytes"] += 8 * w * self.m
                self._io["write_s"] += time.perf_counter() - t0

            fut = self.wpool.submit(work)
            self.wfut[slot] = fut
            futs.append(fut)
        return futs

    # -- factorization ---------------------------------------------------------------------
    def factorize(self) -> dict:
        import torch

        if self.src is None:
            raise ValueError("factorize needs a source store")
        m, n, nb, lda = self.m, self.n, self.nb, self.lda
        d = torch.empty((self.sp_cols, lda), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pending: list = []
        chk = _native.check
        for c0 in range(0, n, self.sp_cols):
            c1 = min(n, c0 + self.sp_cols)
            w = c1 - c0
            d[:w].zero_()

            def load(item, buf, c0=c0):
                k, kw = item[0], item[3]
                d[k * nb - c0:k * nb - c0 + kw, :m].copy_(buf[:kw, :m])

            self._stream(self.src, [(k, 0, None, min(nb, n - k * nb))
                                    for k in range(c0 // nb, -(-c1 // nb))], load)
            # reflectors of earlier super-panels must be on disk before they are streamed
            for f in pending:
                f.result()
            pending = []

            def apply(item, buf, w=w):
                k, np_ = item[0], item[4]
                self._apply_block(k, np_, buf, k * nb, d, k * nb, w)

            self._stream(self.dst, [(k, k * nb, None, self._block_width(k, np_), np_)
                                    for k, np_ in self._blocks(c0 // nb)], apply)
            # right-looking inside the super-panel (the device driver)
            self._factor_in_core(d, c0, w)
            pending = self._write_superpanel(d, c0, c1)
        for f in pending:
            f.result()
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
        self.stats = {"seconds": secs, "tflops": fl / secs / 1e12,
                      "super_panels": -(-n // self.sp_cols), "super_panel_cols": self.sp_cols,
                      **self._io}
        return self.stats

    # -- solve --------------------------------------------------------------------------------
    def rdiag(self) -> np.ndarray:
        """Diagonal of R from the diagonal blocks of the factored store."""
        nb = self.nb
        out = np.empty(self.n)
        blk = np.zeros((nb, nb), order="F")
        for k in range(self.npan):
            j0 = k * nb
            w = min(nb, self.n - j0)
            buf = np.zeros((j0 + w, w), order="F")
            self.dst.read_columns(j0, w, j0, buf, j0 + w)
            out[j0:j0 + w] = np.diag(buf[j0:j0 + w, :w])
        del blk
        return out

    def solve(self, b_dev, report_block: int | None = None):
        """X (device (S, n)) and ||(Q^T b_j)[n:m]|| for b_dev (S, lda) device
        right-hand sides; the factors are streamed from the factored store."""
        import torch

        m, n, nb, lda = self.m, self.n, self.nb, self.lda
        diag = self.rdiag()
        block = int(report_block or n)
        bad = np.flatnonzero(~(np.abs(diag) >= 1e-300))
        if bad.size:
            t = bad.max() // block
            raise SingularMatrixError(int(next(i for i in bad if i // block == t)))
        s = b_dev.shape[0]
        y = b_dev.clone()
        chk = _native.check

        def apply(item, buf):
            k, np_ = item[0], item[4]
            self._apply_block(k, np_, buf, k * nb, y, k * nb, s)

        self._stream(self.dst, [(k, k * nb, None, self._block_width(k, np_), np_)
                                for k, np_ in self._blocks(self.npan)], apply)
        resid = torch.linalg.norm(y[:, n:m], dim=1)

        def back(item, buf):
            k = item[0]
            i0 = k * nb
            bs = min(nb, n - i0)
            chk(self.lib.qrb_op_trsm_upper(_p(buf, i0), lda, bs, 16, _p(y, i0), lda, s, None),
                "qrb_op_trsm_upper")
            if i0 > 0:
                chk(self.lib.qrb_op_gemm_nn_sub(_p(buf), lda, _p(y, i0), lda, _p(y), lda, i0, s,
                                                bs, None), "qrb_op_gemm_nn_sub")

        self._stream(self.dst, [(k, 0, k * nb + min(nb, n - k * nb), min(nb, n - k * nb))
                                for k in range(self.npan - 1, -1, -1)], back)
        torch.cuda.synchronize()
        return y[:, :n], resid
