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


class _StagedFactors:
    """State and steps shared by the host- and disk-staged engines: per-panel T
    and tau, the merged pair reflectors, the in-core super-panel factorization
    and the reflector block schedule of the left-looking stream.  Subclasses
    set lib, m, n, nb, lda, npan, device, t_all, t2_all, pair_valid, tau."""

    def _init_factors(self, dev) -> None:
        import torch

        nb, w2 = self.nb, 2 * self.nb
        self.device = torch.cuda.current_device()
        self.t_all = torch.zeros((self.npan * nb, nb), dtype=torch.float64, device=dev)
        self.t2_all = torch.zeros((max(1, self.npan // 2) * w2, w2), dtype=torch.float64,
                                  device=dev)
        self.pair_valid = np.zeros(max(1, self.npan // 2), dtype=bool)
        self.tau = torch.zeros(self.npan * nb, dtype=torch.float64, device=dev)

    @staticmethod
    def super_panel_cols(n: int, nb: int, lda: int, budget_bytes: int) -> int:
        """Columns of a super-panel: a whole number of panel pairs that fits the
        HBM budget next to two pair-wide reflector staging buffers."""
        w2 = 2 * nb
        col_bytes = 8 * lda
        sp_pairs = max(1, (int(budget_bytes) - 2 * col_bytes * w2) // (col_bytes * w2))
        return min(n, sp_pairs * w2)

    def _blocks(self, upto: int):
        """Reflector blocks of panels [0, upto): (first panel, panels) -- merged
        pairs where the in-core step formed one, single panels otherwise."""
        k = 0
        while k < upto:
            if k % 2 == 0 and k + 1 < upto and self.pair_valid[k // 2]:
                yield k, 2
                k += 2
            else:
                yield k, 1
                k += 1

    def _block_width(self, k: int, panels: int) -> int:
        return min(panels * self.nb, self.n - k * self.nb)

    def _apply_block(self, k: int, panels: int, v, v_row_off: int, c, c_row_off: int,
                     ncols: int) -> None:
        """C[rows k nb.., :ncols] <- Q_block^T C, V of the block in v (ld lda)."""
        j0 = k * self.nb
        w = self._block_width(k, panels)
        if panels == 2:
            t, ldt = _p(self.t2_all, (k // 2) * 4 * self.nb * self.nb), 2 * self.nb
        else:
            t, ldt = _p(self.t_all, k * self.nb * self.nb), self.nb
        st = self.lib.qrb_op_apply_qt(_p(v, v_row_off), self.lda, self.m - j0, w, t, ldt,
                                      _p(c, c_row_off), self.lda, ncols, None)
        _native.check(st, "qrb_op_apply_qt")

    def _factor_in_core(self, d, c0: int, w: int) -> None:
        """Factor rows c0.., columns [c0, c0 + w) of the super-panel d (device,
        ld lda) in place with the device driver (qrb_factorize on a view handle:
        CholeskyQR2 panels, merged pairs, look-ahead); keep tau, T and the merged
        pair reflectors for the later left-looking streams."""
        nb, w2 = self.nb, 2 * self.nb
        h = ctypes.c_void_p()
        _native.check(self.lib.qrb_create_view(self.device, self.m - c0, w, nb, _p(d, c0),
                                               self.lda, ctypes.byref(h)), "qrb_create_view")
        try:
            rep = _native.QrbReport()
            _native.check(self.lib.qrb_factorize(h, ctypes.byref(rep)), "qrb_factorize")
            k0 = c0 // nb
            _native.check(self.lib.qrb_get_factors(h, _p(self.tau, c0),
                                                   _p(self.t_all, k0 * nb * nb), nb),
                          "qrb_get_factors")
            npairs = (-(-w // nb)) // 2
            if npairs:
                _native.check(self.lib.qrb_get_pair_factors(
                    h, _p(self.t2_all, (c0 // w2) * w2 * w2), w2), "qrb_get_pair_factors")
                pairs_on = _native.get_tuning("outer_panels") != 1  # 0 = auto: pairs
                for p in range(npairs):
                    # qrb_api.cu pair_ok: both panels full and 2nb rows below
                    self.pair_valid[c0 // w2 + p] = (pairs_on and (p + 1) * w2 <= w
                                                     and self.m - c0 - p * w2 >= w2)
        finally:
            self.lib.qrb_destroy(h)


class HostStagedQR(_StagedFactors):
    """QR of an m x n matrix held in a pinned host torch tensor of shape (n, lda)
    (column-major, factored in place), using at most ``budget_bytes`` of HBM for
    the super-panel (plus two pair-wide reflector staging buffers).

    In-core steps run the full device driver (qrb_factorize on a view handle of
    the super-panel: CholeskyQR2 panels, merged panel pairs, look-ahead); the
    left-looking stream applies earlier panels two at a time with their merged
    2nb x 2nb reflectors (qrb_get_pair_factors), K = 2nb GEMMs."""

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
        if self.lda % 2:
            raise ValueError("the host matrix's leading dimension must be even")
        self.npan = -(-n // nb)
        self.sp_cols = self.super_panel_cols(n, nb, self.lda, budget_bytes)
        self._init_factors(torch.device("cuda"))
        self.copy_stream = torch.cuda.Stream()
        self.stats: dict = {}

    # -- helpers --------------------------------------------------------------------
    def _stage_v(self, k: int, width: int, dst, stream) -> None:
        """H2D of reflector columns [k nb, k nb + width) (rows j0..) into dst (ld = lda)."""
        j0 = k * self.nb
        st = self.lib.qrb_copy_2d(_p(dst), self.lda, _p(self.a, j0 + j0 * self.lda), self.lda,
                                  self.m - j0, width, 0, ctypes.c_void_p(stream.cuda_stream))
        _native.check(st, "qrb_copy_2d")

    def _stream_previous(self, c, upto: int, vbufs, col_count: int, row_base=0) -> int:
        """Apply Q_k^T for panels k < upto to the device block c (cols col_count),
        reflectors streamed from the host double-buffered; returns H2D bytes."""
        import torch

        blocks = list(self._blocks(upto))
        if not blocks:
            return 0
        cur = torch.cuda.current_stream()
        done = [torch.cuda.Event(), torch.cuda.Event()]
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        moved = 0
        self.copy_stream.wait_stream(cur)
        with torch.cuda.stream(self.copy_stream):
            k, np_ = blocks[0]
            self._stage_v(k, self._block_width(k, np_), vbufs[0], self.copy_stream)
            ready[0].record(self.copy_stream)
        for i, (k, np_) in enumerate(blocks):
            b = i % 2
            if i + 1 < len(blocks):
                nb_ = (i + 1) % 2
                k1, np1 = blocks[i + 1]
                with torch.cuda.stream(self.copy_stream):
                    if i >= 1:
                        self.copy_stream.wait_event(done[nb_])
                    self._stage_v(k1, self._block_width(k1, np1), vbufs[nb_], self.copy_stream)
                    ready[nb_].record(self.copy_stream)
            cur.wait_event(ready[b])
            self._apply_block(k, np_, vbufs[b], 0, c, row_base + k * self.nb, col_count)
            done[b].record(cur)
            moved += 8 * (self.m - k * self.nb) * self._block_width(k, np_)
        return moved

    # -- factorization ------------------------------------------------------------------
    def factorize(self) -> dict:
        import torch

        m, n, nb, lda = self.m, self.n, self.nb, self.lda
        dev = torch.device("cuda")
        d = torch.empty((self.sp_cols, lda), dtype=torch.float64, device=dev)
        vbufs = [torch.empty((2 * nb, lda), dtype=torch.float64, device=dev) for _ in range(2)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2d = d2h = v_bytes = 0
        in_core_s = 0.0
        for c0 in range(0, n, self.sp_cols):
            c1 = min(n, c0 + self.sp_cols)
            w = c1 - c0
            d[:w].copy_(self.a[c0:c1], non_blocking=True)
            h2d += 8 * w * lda
            # left-looking: every earlier panel's reflectors, streamed from the host
            v_bytes += self._stream_previous(d, c0 // nb, vbufs, w)
            # right-looking inside the super-panel (the device driver)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            self._factor_in_core(d, c0, w)
            in_core_s += time.perf_counter() - t1
            self.a[c0:c1].copy_(d[:w], non_blocking=True)
            d2h += 8 * w * lda
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        del d, vbufs
        fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
        self.stats = {"seconds": secs, "tflops": fl / secs / 1e12, "h2d_bytes": h2d + v_bytes,
                      "d2h_bytes": d2h, "v_stream_bytes": v_bytes,
                      "super_panels": -(-n // self.sp_cols), "super_panel_cols": self.sp_cols,
                      "in_core_s": in_core_s}
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
        vbufs = [torch.empty((2 * nb, lda), dtype=torch.float64, device=dev) for _ in range(2)]
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
