"""Python face of one GPU-resident QR factorization (wraps a ``qrb_handle``).

``QrDevice`` holds the m x n matrix in HBM (column-major, leading dimension
padded to 32), factors it in place with the sm_100a kernels and solves many
right-hand sides against the stored factors.  Host arrays are numpy; device
arrays are torch CUDA tensors holding a column-major matrix as a row-major
tensor of shape ``(cols, ld)`` (see :func:`colmajor`).

There is no CPU path: constructing a ``QrDevice`` without the native library
raises :class:`~paper_1907_01891_b200.errors.NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import SingularMatrixError


def _host_f64_fortran(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


def _host_colmajor(a: np.ndarray) -> tuple[np.ndarray, int]:
    """(array, leading dimension) without copying when `a` is column-contiguous
    with a padded leading dimension (e.g. a row slice of a pinned buffer)."""
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if (a.dtype == np.float64 and a.strides[0] == 8 and a.strides[1] % 8 == 0
            and a.strides[1] // 8 >= a.shape[0]):
        return a, a.strides[1] // 8
    a = np.asfortranarray(a, dtype=np.float64)
    return a, a.shape[0]


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def colmajor(t) -> tuple[int, int, int, int]:
    """(data_ptr, rows, cols, ld) of a torch tensor holding a column-major matrix.

    A column-major ``rows x cols`` matrix with leading dimension ``ld`` is stored
    as a contiguous torch tensor of shape ``(cols, ld)`` (rows = ld unless the
    caller passes a narrower logical row count separately).
    """
    if t.dim() != 2 or not t.is_contiguous():
        raise ValueError("expected a contiguous 2-D tensor of shape (cols, ld)")
    cols, ld = t.shape
    return t.data_ptr(), ld, cols, ld


class QrDevice:
    """One m x n fp64 matrix resident on one GPU, factored with panel width nb."""

    def __init__(self, m: int, n: int, nb: int = 128, device: int = 0):
        if m < n:
            raise ValueError(f"matrix must have rows >= cols, got {m}x{n}")
        self.lib = _native.load()
        self.m, self.n, self.nb, self.device = int(m), int(n), int(nb), int(device)
        h = ctypes.c_void_p()
        _native.check(self.lib.qrb_create(self.device, self.m, self.n, self.nb, ctypes.byref(h)),
                      "qrb_create")
        self._h = h
        self.npanels = -(-self.n // self.nb)
        self.last_report: dict = {}

    @classmethod
    def view(cls, t, m: int, n: int, nb: int = 128, device: int = 0) -> "QrDevice":
        """A handle over the caller's device matrix ``t`` (torch tensor (cols, ld),
        column-major m x n with ld even, cols >= n), factored / solved in place
        without a library-owned copy (qrb_create_view); ``t`` is kept alive."""
        if m < n:
            raise ValueError(f"matrix must have rows >= cols, got {m}x{n}")
        ptr, _, cols, ld = colmajor(t)
        if cols < n or ld < m:
            raise ValueError(f"view of {cols} x {ld} storage cannot hold a {m} x {n} matrix")
        self = cls.__new__(cls)
        self.lib = _native.load()
        self.m, self.n, self.nb, self.device = int(m), int(n), int(nb), int(device)
        h = ctypes.c_void_p()
        _native.check(self.lib.qrb_create_view(self.device, self.m, self.n, self.nb,
                                                ctypes.c_void_p(ptr), ld, ctypes.byref(h)),
                      "qrb_create_view")
        self._h = h
        self._storage = t
        self.npanels = -(-self.n // self.nb)
        self.last_report = {}
        return self

    # -- lifecycle ----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.qrb_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- matrix in / out -----------------------------------------------------
    def set_matrix(self, a, col0: int = 0) -> None:
        """Upload columns [col0, col0 + a.shape[1]) from a host array (m x k).
        Column-contiguous arrays with a padded leading dimension (e.g. a view
        of a pinned buffer) are copied without staging."""
        a, ld = _host_colmajor(a)
        if a.shape[0] != self.m:
            raise ValueError(f"expected {self.m} rows, got {a.shape[0]}")
        _native.check(self.lib.qrb_set_matrix(self._h, col0, a.shape[1], _ptr(a), ld, 0),
                      "qrb_set_matrix")

    def set_stream(self, stream_handle: int | None) -> None:
        """Enqueue this handle's work on a CUDA stream (int handle, e.g.
        ``torch.cuda.current_stream().cuda_stream``); None = the handle's own
        blocking stream (ordered with the legacy default stream)."""
        _native.check(self.lib.qrb_set_stream(self._h, ctypes.c_void_p(stream_handle or 0)),
                      "qrb_set_stream")

    def set_profiling(self, on: bool = True) -> None:
        _native.check(self.lib.qrb_set_profiling(self._h, int(bool(on))), "qrb_set_profiling")

    def set_matrix_device(self, t, col0: int = 0) -> None:
        """Copy columns from a torch CUDA tensor of shape (k, ld) (column-major m x k)."""
        ptr, _, cols, ld = colmajor(t)
        _native.check(self.lib.qrb_set_matrix(self._h, col0, cols, ctypes.c_void_p(ptr), ld, 1),
                      "qrb_set_matrix")

    def get_matrix(self, col0: int = 0, ncols: int | None = None) -> np.ndarray:
        """Factored storage (R on/above the diagonal, reflectors below), m x ncols."""
        ncols = self.n - col0 if ncols is None else ncols
        out = np.empty((self.m, ncols), dtype=np.float64, order="F")
        _native.check(self.lib.qrb_get_matrix(self._h, col0, ncols, _ptr(out), self.m, 0),
                      "qrb_get_matrix")
        return out

    def get_matrix_async(self, col0: int, ncols: int, dst: np.ndarray, stream_handle: int) -> None:
        """Columns [col0, col0 + ncols) into the column-major host array dst
        (m x ncols view, page-locked for a real async copy) on a caller stream,
        without waiting (qrb_get_matrix_async)."""
        dst, ld = _host_colmajor(dst)
        _native.check(self.lib.qrb_get_matrix_async(self._h, int(col0), int(ncols), _ptr(dst), ld,
                                                    ctypes.c_void_p(stream_handle)),
                      "qrb_get_matrix_async")

    def get_matrix_device(self, t, col0: int = 0) -> None:
        """Copy factored columns [col0, col0 + k) into a torch CUDA tensor of
        shape (k, ld) (column-major m x k, ld >= m), device to device."""
        ptr, _, cols, ld = colmajor(t)
        _native.check(self.lib.qrb_get_matrix(self._h, col0, cols, ctypes.c_void_p(ptr), ld, 1),
                      "qrb_get_matrix")

    def r_factor(self) -> np.ndarray:
        return np.triu(self.get_matrix()[: self.n, :])

    def rdiag(self) -> np.ndarray:
        d = np.empty(self.n)
        _native.check(self.lib.qrb_get_rdiag(self._h, _ptr(d)), "qrb_get_rdiag")
        return d

    def factors(self) -> tuple[np.ndarray, np.ndarray]:
        """(tau[n], T stacked as nb x npanels*nb)."""
        tau = np.empty(self.n)
        t = np.empty((self.nb, self.npanels * self.nb), order="F")
        _native.check(self.lib.qrb_get_factors(self._h, _ptr(tau), _ptr(t), self.nb),
                      "qrb_get_factors")
        return tau, t

    def set_factors(self, tau: np.ndarray, t: np.ndarray) -> None:
        tau = np.ascontiguousarray(tau, dtype=np.float64)
        t = np.asfortranarray(t, dtype=np.float64)
        if tau.shape != (self.n,) or t.shape != (self.nb, self.npanels * self.nb):
            raise ValueError("factor shapes do not match this handle")
        _native.check(self.lib.qrb_set_factors(self._h, _ptr(tau), _ptr(t), self.nb),
                      "qrb_set_factors")

    def set_pair_factors(self, t2) -> None:
        """Merged 2nb x 2nb reflectors of the panel pairs (after set_factors):
        a torch CUDA tensor (npairs, 2nb, 2nb) -- pair p's block column-major in
        t2[p] -- so the solve skips merging them (qrb_set_pair_factors)."""
        w2 = 2 * self.nb
        if t2.dim() != 3 or tuple(t2.shape[1:]) != (w2, w2) or not t2.is_contiguous():
            raise ValueError("expected a contiguous (npairs, 2nb, 2nb) tensor")
        _native.check(self.lib.qrb_set_pair_factors(self._h, ctypes.c_void_p(t2.data_ptr()), w2),
                      "qrb_set_pair_factors")

    # -- compute --------------------------------------------------------------
    def factorize(self) -> dict:
        rep = _native.QrbReport()
        _native.check(self.lib.qrb_factorize(self._h, ctypes.byref(rep)), "qrb_factorize")
        self.last_report = rep.as_dict()
        return self.last_report

    def factorize_host(self, a, chunk_cols: int = 0) -> dict:
        """set_matrix(host A) + factorize with the PCIe copy overlapped: A is
        copied in column chunks and each chunk is factored left-looking as soon
        as it lands (qrb_factorize_host).  Pass pinned memory for real overlap."""
        a, lda = _host_colmajor(a)
        if a.shape != (self.m, self.n):
            raise ValueError(f"matrix must be {self.m}x{self.n}, got {a.shape}")
        rep = _native.QrbReport()
        _native.check(self.lib.qrb_factorize_host(self._h, _ptr(a), lda, int(chunk_cols),
                                                  ctypes.byref(rep)), "qrb_factorize_host")
        self.last_report = rep.as_dict()
        return self.last_report

    def factorize_host_gated(self, a, chunk_cols: int, ready: np.ndarray,
                             input_gbps: float = 0.0, progress: np.ndarray | None = None) -> dict:
        """factorize_host while another thread is still filling ``a``: chunk c
        (columns [c*chunk_cols, ...)) is copied once ready[c] > 0 (ready[c] < 0
        aborts).  ``a`` and ``ready`` must be page-locked (``PinnedHostArray``)
        for the copies to overlap; the call releases the GIL while it waits.
        ``progress`` (page-locked int64[1]): kept at the number of leading
        columns whose factored values are final (stream them out with
        ``get_matrix_async`` while the call runs)."""
        a, lda = _host_colmajor(a)
        if a.shape != (self.m, self.n):
            raise ValueError(f"matrix must be {self.m}x{self.n}, got {a.shape}")
        if ready.dtype != np.int32 or ready.size < -(-self.n // chunk_cols):
            raise ValueError("ready must be an int32 array with one flag per chunk")
        rep = _native.QrbReport()
        prog = _ptr(progress) if progress is not None else ctypes.c_void_p(0)
        _native.check(self.lib.qrb_factorize_host_gated(self._h, _ptr(a), lda, int(chunk_cols),
                                                        _ptr(ready), float(input_gbps), prog,
                                                        ctypes.byref(rep)),
                      "qrb_factorize_host_gated")
        self.last_report = rep.as_dict()
        return self.last_report

    def solve(self, b, report_block: int | None = None, want_resid: bool = True, out=None):
        """X = R^-1 (Q^T B)[:n] for host B (m x nrhs); returns (X, resid, report).
        ``out`` may be a preallocated (n x nrhs) column-contiguous host array."""
        b, ldb = _host_colmajor(b)
        if b.shape[0] != self.m:
            raise ValueError(f"right-hand side has {b.shape[0]} rows, expected {self.m}")
        nrhs = b.shape[1]
        if out is None:
            x = np.empty((self.n, nrhs), order="F")
            ldx = self.n
        else:
            x, ldx = _host_colmajor(out)
            if x is not out or x.shape != (self.n, nrhs):
                raise ValueError("out must be a column-contiguous (n x nrhs) float64 array")
        resid = np.empty(nrhs) if want_resid else None
        rep = _native.QrbReport()
        st = self.lib.qrb_solve(self._h, _ptr(b), ldb, nrhs, _ptr(x), ldx,
                                _ptr(resid) if want_resid else None, 0,
                                int(report_block or self.n), ctypes.byref(rep))
        st = _native.check(st, "qrb_solve")
        if st > 0:
            raise SingularMatrixError(st - 1)
        self.last_report = rep.as_dict()
        return x, resid, self.last_report

    def solve_device(self, b_t, x_t, resid_t=None, report_block: int | None = None) -> dict:
        """Device-resident solve: b_t (nrhs, ldb) and x_t (nrhs, ldx) torch CUDA tensors."""
        bp, _, nrhs, ldb = colmajor(b_t)
        xp, _, nrhs2, ldx = colmajor(x_t)
        if nrhs2 != nrhs or ldb < self.m or ldx < self.n:
            raise ValueError("solve_device: shape mismatch")
        rp = ctypes.c_void_p(resid_t.data_ptr()) if resid_t is not None else None
        rep = _native.QrbReport()
        st = self.lib.qrb_solve(self._h, ctypes.c_void_p(bp), ldb, nrhs, ctypes.c_void_p(xp), ldx,
                                rp, 1, int(report_block or self.n), ctypes.byref(rep))
        st = _native.check(st, "qrb_solve")
        if st > 0:
            raise SingularMatrixError(st - 1)
        self.last_report = rep.as_dict()
        return self.last_report


class PinnedHostArray:
    """A numpy array in page-locked host memory (cudaHostRegister on a numpy
    allocation: exact size -- torch's pinned allocator rounds requests up to a
    power of two, 64 GB for config 3's 36 GB).  ``.array`` is the array; the
    registration is dropped by ``close()`` / garbage collection."""

    def __init__(self, shape, dtype=np.float64):
        import torch
        self.array = np.empty(shape, dtype=dtype)
        self._cudart = torch.cuda.cudart()
        self._ptr = self.array.ctypes.data
        rc = self._cudart.cudaHostRegister(self._ptr, max(self.array.nbytes, 1), 2)  # Mapped
        if int(rc) != 0:
            raise MemoryError(f"cudaHostRegister of {self.array.nbytes} bytes failed ({rc})")
        self._registered = True

    def close(self) -> None:
        if getattr(self, "_registered", False):
            self._cudart.cudaHostUnregister(self._ptr)
            self._registered = False

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def launch_count() -> int:
    """Kernels launched by libqrb200 in this process so far."""
    return int(_native.load().qrb_launch_count())
