"""ctypes binding of the sm_100a library ``libqrb200.so`` (include/qrb200.h).

This is the only way the package reaches the GPU: there is no CPU fallback.
If the shared library is missing or cannot be loaded, every product entry
point raises :class:`NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NativeUnavailableError

_LIB_PATH = Path(os.environ.get("QRB_LIB_PATH") or
                 Path(__file__).resolve().parent / "_lib" / "libqrb200.so")  # override: A/B builds

c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_dbl_p = ctypes.POINTER(ctypes.c_double)
c_void_p = ctypes.c_void_p

QRB_OK = 0
QRB_EARG = -1
QRB_ECUDA = -2
QRB_ENOMEM = -3
QRB_ENONFINITE = -4
QRB_ESTATE = -5
QRB_EUNSUPPORTED = -6


KERNEL_NAMES = ("panel", "gemm_tn", "gemm_tt", "gemm_nn", "trsm", "gemm_nn_capped", "k6", "k7")


class QrbKernelStat(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double), ("flops", ctypes.c_double),
                ("bytes", ctypes.c_double), ("launches", c_i64)]


class QrbReport(ctypes.Structure):
    """Mirror of ``qrb_report`` (include/qrb200.h)."""

    _fields_ = [
        ("total_ms", ctypes.c_double),
        ("panel_ms", ctypes.c_double),
        ("update_ms", ctypes.c_double),
        ("trsm_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("flops", ctypes.c_double),
        ("kernel_launches", c_i64),
        ("h2d_bytes", c_i64),
        ("d2h_bytes", c_i64),
        ("kernels", QrbKernelStat * 8),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_ if name != "kernels"}
        d["kernels"] = {KERNEL_NAMES[i]: {"ms": k.ms, "flops": k.flops, "bytes": k.bytes,
                                          "launches": int(k.launches)}
                        for i, k in enumerate(self.kernels) if k.launches}
        return d


# exported symbol -> (restype, argtypes); the list IS the C ABI of include/qrb200.h
SIGNATURES = {
    "qrb_version": (c_int, []),
    "qrb_last_error": (ctypes.c_char_p, []),
    "qrb_device_count": (c_int, [ctypes.POINTER(c_int)]),
    "qrb_set_device": (c_int, [c_int]),
    "qrb_create": (c_int, [c_int, c_i64, c_i64, c_int, ctypes.POINTER(c_void_p)]),
    "qrb_create_view": (c_int, [c_int, c_i64, c_i64, c_int, c_void_p, c_i64,
                                ctypes.POINTER(c_void_p)]),
    "qrb_destroy": (c_int, [c_void_p]),
    "qrb_set_matrix": (c_int, [c_void_p, c_i64, c_i64, c_void_p, c_i64, c_int]),
    "qrb_get_matrix": (c_int, [c_void_p, c_i64, c_i64, c_void_p, c_i64, c_int]),
    "qrb_set_profiling": (c_int, [c_void_p, c_int]),
    "qrb_set_stream": (c_int, [c_void_p, c_void_p]),
    "qrb_factorize": (c_int, [c_void_p, ctypes.POINTER(QrbReport)]),
    "qrb_factorize_host": (c_int, [c_void_p, c_void_p, c_i64, c_i64, ctypes.POINTER(QrbReport)]),
    "qrb_factorize_host_gated": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p,
                                         ctypes.c_double, c_void_p, ctypes.POINTER(QrbReport)]),
    "qrb_get_matrix_async": (c_int, [c_void_p, c_i64, c_i64, c_void_p, c_i64, c_void_p]),
    "qrb_get_factors": (c_int, [c_void_p, c_void_p, c_void_p, c_i64]),
    "qrb_get_pair_factors": (c_int, [c_void_p, c_void_p, c_i64]),
    "qrb_set_pair_factors": (c_int, [c_void_p, c_void_p, c_i64]),
    "qrb_set_factors": (c_int, [c_void_p, c_void_p, c_void_p, c_i64]),
    "qrb_solve": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_i64, c_void_p, c_int,
                          c_i64, ctypes.POINTER(QrbReport)]),
    "qrb_get_rdiag": (c_int, [c_void_p, c_void_p]),
    "qrb_op_panel": (c_int, [c_void_p, c_i64, c_i64, c_i64, c_void_p, c_void_p, c_i64, c_void_p]),
    "qrb_op_apply_qt": (c_int, [c_void_p, c_i64, c_i64, c_i64, c_void_p, c_i64, c_void_p, c_i64,
                                c_i64, c_void_p]),
    "qrb_op_panel_block": (c_int, [c_void_p, c_i64, c_i64, c_i64, c_int, c_void_p, c_void_p,
                                   c_void_p, c_i64, c_void_p, c_int]),
    "qrb_op_apply_qt_begin": (c_int, [c_void_p, c_i64, c_i64, c_i64, c_void_p, c_i64, c_void_p,
                                      c_i64, c_i64, c_void_p]),
    "qrb_op_apply_qt_cols": (c_int, [c_void_p, c_i64, c_i64, c_i64, c_void_p, c_i64, c_i64, c_i64,
                                     c_void_p]),
    "qrb_op_apply_qt_td": (c_int, [c_void_p, c_i64, c_i64, c_i64, c_void_p, c_i64, c_void_p,
                                   c_i64, c_void_p, c_i64, c_i64, c_void_p]),
    "qrb_op_gemm_nn_sub": (c_int, [c_void_p, c_i64, c_void_p, c_i64, c_void_p, c_i64, c_i64,
                                   c_i64, c_i64, c_void_p]),
    "qrb_op_gemm_tn": (c_int, [c_void_p, c_i64, c_void_p, c_i64, c_void_p, c_i64, c_i64, c_i64,
                               c_i64, c_int, c_int, c_int, c_void_p]),
    "qrb_op_trsm_upper": (c_int, [c_void_p, c_i64, c_i64, c_int, c_void_p, c_i64, c_i64,
                                  c_void_p]),
    "qrb_siddon_densify": (c_int, [c_void_p, c_i64, c_i64, c_int, c_void_p, c_i64, c_int, c_int,
                                   c_int, c_i64, c_void_p]),
    "qrb_copy_2d": (c_int, [c_void_p, c_i64, c_void_p, c_i64, c_i64, c_i64, c_int, c_void_p]),
    "qrb_launch_count": (c_i64, []),
    "qrb_release_workspace": (c_int, []),
    "qrb_set_tuning": (c_int, [ctypes.c_char_p, c_i64]),
    "qrb_get_tuning": (c_int, [ctypes.c_char_p, ctypes.POINTER(c_i64)]),
}

_lib = None
_load_error: str | None = None


def library_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = False) -> ctypes.CDLL:
    """Load libqrb200.so (optionally building it first)."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if build_if_missing and not _LIB_PATH.exists():
        from . import build as _build

        _build.build()
    if not _LIB_PATH.exists():
        _load_error = f"{_LIB_PATH} not built (run paper_1907_01891_b200.build.build())"
        raise NativeUnavailableError(_load_error)
    try:
        lib = ctypes.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    except OSError as exc:
        _load_error = f"cannot load {_LIB_PATH}: {exc}"
        raise NativeUnavailableError(_load_error) from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    lib = load()
    msg = lib.qrb_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(status: int, what: str) -> int:
    """Raise on negative status; positive (singular column + 1) is returned."""
    if status < 0:
        from .errors import GpuError, KernelInputError

        msg = f"{what} failed (status {status}): {last_error()}"
        if status == QRB_ENONFINITE:
            raise KernelInputError(msg)
        raise GpuError(msg)
    return status


def set_tuning(key: str, value: int) -> None:
    """Process-wide knob of the native library (qrb_set_tuning)."""
    check(load().qrb_set_tuning(key.encode(), int(value)), f"qrb_set_tuning({key})")


def get_tuning(key: str) -> int:
    out = c_i64(0)
    check(load().qrb_get_tuning(key.encode(), ctypes.byref(out)), f"qrb_get_tuning({key})")
    return int(out.value)
