"""B200-native (sm_100a) drop-in for the hot path of ``oocqr`` (arXiv 1907.01891):
dense blocked Householder QR of the CT system matrix, Q^T applied to many
sinograms and the R back-substitution, behind the reference's own
``factorize`` / ``solve`` API (pkg/src/oocqr/__init__.py:9-23).

All arithmetic runs in ``_lib/libqrb200.so`` (hand-written sm_100a CUDA, C ABI
in ``include/qrb200.h``); there is no CPU fallback.
"""

from .errors import (CacheCapacityError, CorruptTileError, GpuError, KernelInputError,
                     ManifestError, MissingFactorsError, NativeUnavailableError,
                     SingularMatrixError, TaskIoError)
from .tile_store import TileCache, TiledMatrix, TileId, gather_matrix, scatter_matrix
from .task_engine import EngineConfig, QrFactors, RunReport, factorize, solve

__version__ = "0.1.0"

__all__ = [
    "TileCache",
    "TiledMatrix",
    "TileId",
    "EngineConfig",
    "RunReport",
    "QrFactors",
    "factorize",
    "solve",
    "gather_matrix",
    "scatter_matrix",
    "KernelInputError",
    "SingularMatrixError",
    "TaskIoError",
    "MissingFactorsError",
    "ManifestError",
    "CorruptTileError",
    "CacheCapacityError",
    "NativeUnavailableError",
    "GpuError",
    "__version__",
]
