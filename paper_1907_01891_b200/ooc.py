"""Host-staged (out-of-HBM) QR and solve: matrices larger than the HBM budget.

BASELINE config 4 (270000 x 262144 fp64 = 566 GB) exceeds a B200's 180 GB at
fewer than 4 GPUs.  The reference's answer to "larger than memory" is its
out-of-core tile engine: left-looking by tile columns so each produced tile is
written once (task_engine.py:4-9, 187-217), a bounded cache
and one prefetch thread (task_engine.py:330-474).  The B200 version keeps the
matrix in pinned host memory and works left-looking by *super-panels* that fit
the HBM budget:

  for each super-panel S (as many panels of nb columns as fit):
      H2D  S                                          (once)
      for every earlier panel k:  stream V_k H2D (double-buffered on a copy
          stream, overlapping the previous apply) and apply Q_k^T to S
          (the DMMA block-reflector kernels)
      factor S in core: right-looking panels + trailing updates inside S
      D2H  S                                          (once)

so every column block crosses PCIe twice and the reflectors are re-streamed
(#super-panels / 2) times on average, while all arithmetic stays on the GPU.
T factors and tau (small) stay resident on the device.  The solve streams the
reflector panels once per right-hand-side batch for Q^T B and the R block
columns once for the back-substitution.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native
from .errors import SingularMatrixError


def _p(t, off: int = 0) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() + 8 * off)


class HostStagedQR:
    """QR of an m x n matrix held in a pinned host torch tensor of shape (n, lda)
    (column-major, factored in place), using at most ``budget_bytes`` of HBM for
    the super-panel (plus two reflector staging buffers)."""

    def __init__(self, a_host, m: int, n: int, nb: int = 128, budget_bytes: int = 32 << 30):
        import torch

        if m < n:
            raise ValueError(f"matrix must have rows >= cols, got {m}x{n}")
        if not a_host.is_pinned():
            raise ValueError("a_host must be a pinned host tensor (torch.empty(..., pin_memory=True))")
        self.lib = _native.load()
        self.a = a_host
        self.m, self.n, self.nb = m, n, nb
        self.lda = a_host.shape[1]
        self.npan = -(-n // nb)
        col_bytes = 8 * self.lda
        stage_bytes = 2 * col_bytes * nb
        sp_panels = max(1, (int(budget_bytes) - stage_bytes) // (col_bytes * nb))
        self.sp_cols = min(n, sp_panels * nb)
        dev = torch.device("cuda")
        self.t_all = torch.zeros((self.npan * nb, nb), dtype=torch.float64, device=dev)
        self.tau = torch.zeros(self.npan * nb, dtype=torch.float64, device=dev)
        self.copy_stream = torch.cuda.Stream()
        self.stats: dict = {}

    # -- helpers --------------------------------------------------------------------
    def _stage_v(self, k: int, dst, stream) -> None:
        """H2D of reflector panel k (rows j0.., pw columns) into dst (ld = lda)."""
        j0 = k * self.nb
        pw = min(self.nb, self.n - j0)
        st = self.lib.qrb_copy_2d(_p(dst), self.lda, _p(self.a, j0 + j0 * self.lda), self.lda,
                                  self.m - j0, pw, 0, ctypes.c_void_p(stream.cuda_stream))
        _native.check(st, "qrb_copy_2d")

    def _apply(self, k: int, v, c, c_row_off: int, ncols: int) -> None:
        j0 = k * self.nb
        pw = min(self.nb, self.n - j0)
        st = self.lib.qrb_op_apply_qt(_p(v), self.lda, self.m - j0, pw,
                                      _p(self.t_all, k * self.nb * self.nb), self.nb,
                                      _p(c, c_row_off), self.lda, ncols, None)
        _native.check(st, "qrb_op_apply_qt")

    def _stream_previous(self, c, upto: int, vbufs, col_count: int, row_base=0) -> None:
        """Apply Q_k^T for k < upto to the device block c (cols col_count)."""
        import torch

        cur = torch.cuda.current_stream()
        done = [torch.cuda.Event(), torch.cuda.Event()]
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        if upto <= 0:
            return
        self.copy_stream.wait_stream(cur)
        with torch.cuda.stream(self.copy_stream):
            self._stage_v(0, vbufs[0], self.copy_stream)
            ready[0].record(self.copy_stream)
        for k in range(upto):
            b = k % 2
            if k + 1 < upto:
                nb_ = (k + 1) % 2
                with torch.cuda.stream(self.copy_stream):
                    if k >= 1:
                        self.copy_stream.wait_event(done[nb_])
                    self._stage_v(k + 1, vbufs[nb_], self.copy_stream)
                    ready[nb_].record(self.copy_stream)
            cur.wait_event(ready[b])
            self._apply(k, vbufs[b], c, row_base + k * self.nb, col_count)
            done[b].record(cur)

    # -- factorization ------------------------------------------------------------------
    def factorize(self) -> dict:
        import torch

        m, n, nb, lda = self.m, self.n, self.nb, self.lda
        dev = torch.device("cuda")
        d = torch.empty((self.sp_cols, lda), dtype=torch.float64, device=dev)
        vbufs = [torch.empty((nb, lda), dtype=torch.float64, device=dev) for _ in range(2)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for c0 in range(0, n, self.sp_cols):
            c1 = min(n, c0 + self.sp_cols)
            w = c1 - c0
            d[:w].copy_(self.a[c0:c1], non_blocking=True)
            h2d += 8 * w * lda
            # left-looking: every earlier panel's reflectors, streamed from the host
            k0 = c0 // nb
            self._stream_previous(d, k0, vbufs, w)
            h2d += sum(8 * (m - k * nb) * min(nb, n - k * nb) for k in range(k0))
            # right-looking inside the super-panel
            for k in range(k0, -(-c1 // nb)):
                j0 = k * nb
                pw = min(nb, n - j0)
                lc = j0 - c0
                st = self.lib.qrb_op_panel(_p(d, j0 + lc * lda), lda, m - j0, pw,
                                           _p(self.tau, j0), _p(self.t_all, k * nb * nb), nb,
                                           None)
                _native.check(st, "qrb_op_panel")
                rest = w - (lc + pw)
                if rest > 0:
                    st = self.lib.qrb_op_apply_qt(_p(d, j0 + lc * lda), lda, m - j0, pw,
                                                  _p(self.t_all, k * nb * nb), nb,
                                                  _p(d, j0 + (lc + pw) * lda), lda, rest, None)
                    _native.check(st, "qrb_op_apply_qt")
            self.a[c0:c1].copy_(d[:w], non_blocking=True)
            d2h += 8 * w * lda
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
        self.stats = {"seconds": secs, "tflops": fl / secs / 1e12, "h2d_bytes": h2d,
                      "d2h_bytes": d2h, "super_panels": -(-n // self.sp_cols),
                      "super_panel_cols": self.sp_cols}
        return self.stats

    # -- solve ------------------------------------------------------------------------------
    def solve(self, b_dev, report_block: int | None = None):
        """X (n x S, device tensor (S, n)) for b_dev (S, lda) device right-hand sides;
        returns (x, resid) with resid_j = ||(Q^T b_j)[n:m]||."""
        import torch

        m, n, nb, lda = self.m, self.n, self.nb, self.lda
        diag = torch.diagonal(self.a[:, :n]).clone().numpy() if n else np.zeros(0)
        block = int(report_block or n)
        bad = np.flatnonzero(~(np.abs(diag) >= 1e-300))
        if bad.size:
            t = bad.max() // block
            first = next(i for i in bad if i // block == t)
            raise SingularMatrixError(int(first))
        s = b_dev.shape[0]
        y = b_dev.clone()
        dev = torch.device("cuda")
        vbufs = [torch.empty((nb, lda), dtype=torch.float64, device=dev) for _ in range(2)]
        self._stream_previous(y, self.npan, vbufs, s)
        resid = torch.linalg.norm(y[:, n:m], dim=1)
        # back substitution, bottom-up block columns of R streamed from the host
        rbuf = torch.empty((nb, lda), dtype=torch.float64, device=dev)
        for k in range(self.npan - 1, -1, -1):
            i0 = k * nb
            bs = min(nb, n - i0)
            i1 = i0 + bs
            st = self.lib.qrb_copy_2d(_p(rbuf), lda, _p(self.a, i0 * lda), lda, i1, bs, 0, None)
            _native.check(st, "qrb_copy_2d")
            st = self.lib.qrb_op_trsm_upper(_p(rbuf, i0), lda, bs, 16, _p(y, i0), lda, s, None)
            _native.check(st, "qrb_op_trsm_upper")
            if i0 > 0:
                st = self.lib.qrb_op_gemm_nn_sub(_p(rbuf), lda, _p(y, i0), lda, _p(y), lda, i0, s,
                                                 bs, None)
                _native.check(st, "qrb_op_gemm_nn_sub")
        torch.cuda.synchronize()
        return y[:, :n], resid
