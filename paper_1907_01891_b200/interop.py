"""Solve on the GPU against factors produced by the CPU reference.

The reference persists its factorization as two tiled stores -- ``factored``
(R on/above the diagonal, per-tile reflectors below / in the TD tiles) and
``s`` (packed T factors of every tile task) -- plus ``meta.txt`` (rows, cols,
tile_size, inner_block, geometry_hash), task_engine.py:531-594.  Its Q is a
product of per-tile dense and triangle-on-dense reflector blocks, applied in
the order of ``gen_solve_tasks`` (task_engine.py:220-254).

:func:`solve_reference_factors` replays exactly that task order on the GPU:
``apply_left_qt_dense`` through ``qrb_op_apply_qt`` (unit-lower V read in
place), ``apply_left_qt_td`` through ``qrb_op_apply_qt_td``, ``gemm_nn_mo``
through ``qrb_op_gemm_nn_sub`` and ``trsm_lunn`` through ``qrb_op_trsm_upper``
-- all DMMA kernels -- with every right-hand side in one batch (the tile tasks
act column by column, so the RHS block split of the reference does not change
the result).  Tiles live in a padded tile grid in HBM so every tile view is
16-byte aligned (TMA requirement); tile size and inner width must be even.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native
from .errors import MissingFactorsError, SingularMatrixError
from .tile_store import TiledMatrix, TileId


@dataclass
class ReferenceFactors:
    factored: TiledMatrix
    s_store: TiledMatrix
    rows: int
    cols: int
    tile_size: int
    inner_block: int
    geometry_hash: str = ""

    @classmethod
    def load(cls, directory) -> "ReferenceFactors":
        directory = Path(directory)
        meta = directory / "meta.txt"
        if not meta.is_file():
            raise MissingFactorsError(f"no factorization at {directory}")
        fields = {}
        for line in meta.read_text().splitlines():
            if line.strip():
                k, v = line.split(None, 1)
                fields[k] = v.strip()
        if "algorithm" in fields:
            raise MissingFactorsError(f"{directory} is not a reference (tiled TD) factorization")
        return cls(TiledMatrix.open(directory / "factored"), TiledMatrix.open(directory / "s"),
                   int(fields["rows"]), int(fields["cols"]), int(fields["tile_size"]),
                   int(fields["inner_block"]),
                   "" if fields.get("geometry_hash", "-") == "-" else fields["geometry_hash"])

    def save(self, directory) -> None:
        text = (f"rows {self.rows}\ncols {self.cols}\ntile_size {self.tile_size}\n"
                f"inner_block {self.inner_block}\ngeometry_hash {self.geometry_hash or '-'}\n")
        (Path(directory) / "meta.txt").write_text(text)


def _p(t, off=0):
    return ctypes.c_void_p(t.data_ptr() + 8 * off)


def solve_reference_factors(f: ReferenceFactors, bmat: np.ndarray):
    """X (cols x nrhs, host) = R^-1 (Q^T B)[:cols] with the reference's Q."""
    import torch

    lib = _native.load()
    b, w = f.tile_size, f.inner_block
    if b % 2 or w % 2:
        raise NotImplementedError("GPU interop needs an even tile size and inner block")
    bmat = np.asarray(bmat, dtype=np.float64)
    if bmat.ndim == 1:
        bmat = bmat[:, None]
    if bmat.shape[0] != f.rows:
        raise ValueError(f"right-hand side has {bmat.shape[0]} rows, factors expect {f.rows}")
    p, q = f.factored.grid_rows, -(-f.cols // b)
    nrhs = bmat.shape[1]
    dev = torch.device("cuda")
    ldp = p * b                        # padded tile-grid leading dimension (even)
    fac = torch.zeros((q * b, ldp), dtype=torch.float64, device=dev)   # (cols, ld)
    sfa = torch.zeros((q * b, ldp), dtype=torch.float64, device=dev)
    for k in range(q):
        for i in range(p):
            for store, dst in ((f.factored, fac), (f.s_store, sfa)):
                if store.tile_path(TileId(i, k)).exists():
                    t = store.load_tile(TileId(i, k))          # C-order b x b
                    dst[k * b:(k + 1) * b, i * b:(i + 1) * b] = torch.from_numpy(t.T.copy()).to(dev)
    y = torch.zeros((nrhs, ldp), dtype=torch.float64, device=dev)
    y[:, :f.rows] = torch.from_numpy(np.ascontiguousarray(bmat.T)).to(dev)

    def tile_off(i, k):               # element offset of tile (i, k) in a (cols, ldp) tensor
        return i * b + k * b * ldp

    chk = _native.check
    # Q^T B in the order of gen_solve_tasks (task_engine.py:233-245)
    for k in range(q):
        for j0 in range(0, b, w):
            pw = min(w, b - j0)
            chk(lib.qrb_op_apply_qt(_p(fac, tile_off(k, k) + j0 + j0 * ldp), ldp, b - j0, pw,
                                    _p(sfa, tile_off(k, k) + j0), ldp,
                                    _p(y, k * b + j0), ldp, nrhs, None), "qrb_op_apply_qt")
        for i in range(k + 1, p):
            chk(lib.qrb_op_apply_qt_td(_p(fac, tile_off(i, k)), ldp, b, w,
                                       _p(sfa, tile_off(i, k)), ldp, _p(y, k * b), ldp,
                                       _p(y, i * b), ldp, nrhs, None), "qrb_op_apply_qt_td")
    # bottom-up block back substitution (task_engine.py:246-253)
    for k in range(q - 1, -1, -1):
        for j in range(k + 1, q):
            chk(lib.qrb_op_gemm_nn_sub(_p(fac, tile_off(k, j)), ldp, _p(y, j * b), ldp,
                                       _p(y, k * b), ldp, b, nrhs, b, None), "qrb_op_gemm_nn_sub")
        extent = min(b, f.cols - k * b)
        diag = torch.diagonal(fac[k * b:k * b + extent, k * b:k * b + extent]).cpu().numpy()
        bad = np.flatnonzero(~(np.abs(diag) >= 1e-300))
        if bad.size:
            raise SingularMatrixError(k * b + int(bad[0]))
        chk(lib.qrb_op_trsm_upper(_p(fac, tile_off(k, k)), ldp, extent, 16, _p(y, k * b), ldp,
                                  nrhs, None), "qrb_op_trsm_upper")
        y[:, k * b + extent:(k + 1) * b] = 0.0
    torch.cuda.synchronize()
    return y[:, :f.cols].cpu().numpy().T.copy()


def export_reference_factors(directory, factored: np.ndarray, t_blocks: np.ndarray, nb: int,
                             geometry_hash: str = "") -> ReferenceFactors:
    """Write a GPU factorization as an ``oocqr`` factors directory that the
    reference's own ``solve`` reads (meta.txt, ``factored/``, ``s/``;
    task_engine.py:531-594, storage conventions kernels.py:6-20).

    The GPU factorization is one blocked Householder QR of the whole m x n
    matrix with panel width nb: R on/above the diagonal, unit-lower reflectors
    below it, one nb x nb T per panel, Q = H_0 H_1 ... with H_p = I - V_p T_p
    V_p^T.  In the reference's format that is exactly a ONE-tile factorization
    (tile size b = m rounded up to nb, grid 1 x 1, inner_block = nb): the
    reference's ``comp_dense_qr`` of a single b x b tile is the same panel
    recurrence and stores the same (R, V) in the tile and T_p packed at rows
    p*nb : p*nb + nb, columns 0 : nb of the S tile.  Zero padding rows/columns
    (tile_store.py:186-187) contribute nothing: padded reflector columns have
    T = 0.  A multi-tile-row export is not possible without refactoring: the
    reference's Q is a product of per-tile-pair (TD) reflectors, ours of
    full-height panel reflectors.  The caller's right-hand sides must therefore
    be tiled with the same tile size b (``solve`` checks it).

    factored: m x n (host) as QrDevice.get_matrix() returns it; t_blocks:
    nb x (npanels * nb) as QrDevice.factors()[1] returns it.
    """
    directory = Path(directory)
    factored = np.asarray(factored, dtype=np.float64)
    m, n = factored.shape
    npan = -(-n // nb)
    if t_blocks.shape != (nb, npan * nb):
        raise ValueError(f"T blocks must be {nb} x {npan * nb}, got {t_blocks.shape}")
    b = -(-m // nb) * nb
    directory.mkdir(parents=True, exist_ok=True)
    fac = TiledMatrix.create(m, n, b, directory / "factored")
    s_store = TiledMatrix.create(b, b, b, directory / "s")
    tile = np.zeros((b, b))
    tile[:m, :n] = factored
    fac.store_tile(TileId(0, 0), tile)
    tile[:] = 0.0
    for p in range(npan):
        w = min(nb, n - p * nb)
        tile[p * nb:p * nb + w, :w] = np.triu(t_blocks[:w, p * nb:p * nb + w])
    s_store.store_tile(TileId(0, 0), tile)
    f = ReferenceFactors(fac, s_store, m, n, b, nb, geometry_hash)
    f.save(directory)
    return f
