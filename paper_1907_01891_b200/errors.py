"""Exception types of the drop-in API.

Names, bases and attributes mirror the reference package so that callers'
``except`` clauses keep working:

* ``KernelInputError`` / ``SingularMatrixError``  -- kernels.py:40-52
* ``TaskIoError`` / ``MissingFactorsError``       -- task_engine.py:62-71
* ``ManifestError`` / ``CorruptTileError`` / ``CacheCapacityError`` -- tile_store.py:33-42

Two errors are new: ``NativeUnavailableError`` (the sm_100a library is not
built or cannot load -- the product path never falls back to the CPU) and
``GpuError`` (a CUDA failure inside the library).
"""

from __future__ import annotations


class KernelInputError(ValueError):
    """Shape, finiteness, or structure violation in a kernel input."""


class SingularMatrixError(RuntimeError):
    """Zero (or sub-threshold) diagonal entry met during a triangular solve."""

    def __init__(self, global_column: int):
        self.global_column = int(global_column)
        super().__init__(
            f"singular upper-triangular factor: zero pivot at global column "
            f"{self.global_column}"
        )


class TaskIoError(RuntimeError):
    """Disk failure while staging tiles for a task (``seq`` = task position)."""

    def __init__(self, seq: int, op: str, cause: BaseException):
        self.seq = seq
        super().__init__(f"I/O failure at task seq={seq} ({op}): {cause}")


class MissingFactorsError(RuntimeError):
    """Solve requested against an absent or incomplete factorization."""


class ManifestError(RuntimeError):
    """Missing, malformed, or incompatible matrix manifest."""


class CorruptTileError(RuntimeError):
    """Tile file exists but has the wrong length."""


class CacheCapacityError(RuntimeError):
    """No unpinned tile is available for eviction."""


class NativeUnavailableError(RuntimeError):
    """libqrb200.so is missing or failed to load; there is no CPU fallback."""


class GpuError(RuntimeError):
    """A CUDA call inside libqrb200 failed."""
