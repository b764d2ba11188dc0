"""Drop-in ``factorize`` / ``solve`` (reference task_engine.py:606-685) on the GPU.

The reference stages b x b tiles through a disk-backed LRU cache and runs a
left-looking tile DAG on the CPU (task_engine.py:187-523).  Here the whole
matrix is staged once into HBM (column blocks of tiles map straight onto the
column-major device matrix), factored by ``libqrb200`` with the right-looking
blocked Householder QR, and written back in the reference's ``factored``
convention: R on and above the diagonal, unit-diagonal reflectors below.

Public signatures, argument checks, exception types, the "source A and B are
never modified" contract and the ``out_dir/x`` result store all follow the
reference.  What differs, by design:

* the Q representation: one compact-WY (V, T) pair per panel of ``panel_width``
  columns (classical geqrf) instead of the reference's per-tile TD reflectors +
  packed S tiles.  ``meta.txt`` carries ``algorithm geqrf_cwy`` so neither
  package silently misreads the other's factors; R and every solution agree
  with the reference within the fp64 tolerances of BASELINE.json;
* ``RunReport.task_count`` counts GPU kernel launches and the trace lists the
  stage / compute / write-back phases instead of per-tile tasks.
"""

from __future__ import annotations

import csv
import os
import io
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import dist_api
from .device import PinnedHostArray, QrDevice
from .errors import (CacheCapacityError, CorruptTileError, MissingFactorsError,
                     SingularMatrixError, TaskIoError)
from .tile_store import TiledMatrix, TileId

_META_NAME = "meta.txt"
_T_NAME = "t_factors.f64"
_TAU_NAME = "tau.f64"
ALGORITHM = "geqrf_cwy"


@dataclass
class EngineConfig:
    """Reference knobs (task_engine.py:77-121) plus the GPU ones.

    ``tile_size`` / ``inner_block`` keep their reference meaning for the
    on-disk stores and the API checks; ``panel_width`` is the GPU panel width
    nb (a multiple of 16, <= 128) and ``device`` the CUDA device.  Residency
    tiers: a matrix that fits ``hbm_budget_bytes`` is factored in HBM; one that
    does not but fits ``cache_budget_bytes`` (the reference's RAM budget) is
    pinned in host memory and streamed super-panel by super-panel (ooc.py);
    anything larger streams panel by panel from the tile files on disk
    (disk_ooc.py), the reference's own out-of-core regime.
    """

    tile_size: int = 10240
    inner_block: int = 128
    cache_budget_bytes: int = 32 * 2**30
    mode: str = "sequential"
    compute_workers: int = 1
    io_agents: int = 1
    prefetch_depth: int = 2
    panel_width: int = 128
    device: int = 0
    hbm_budget_bytes: int = 0  # 0 = 85% of free HBM; above it A is host-staged (ooc.py)
    # GPUs (= ranks of the torch.distributed process group, one process per GPU,
    # every rank calling factorize/solve with the same arguments -- dist_api.py):
    # 0 = the initialized process group's size (1 without one), 1 = this process's
    # GPU only, N > 1 = require a group of N ranks
    world_size: int = 0

    def validate(self) -> "EngineConfig":
        if self.tile_size < 1:
            raise ValueError(f"tile_size must be >= 1, got {self.tile_size}")
        if not 1 <= self.inner_block <= self.tile_size:
            raise ValueError(f"inner_block must be in [1, tile_size], got {self.inner_block}")
        if self.mode not in ("sequential", "overlapped"):
            raise ValueError(f"mode must be sequential or overlapped, got {self.mode!r}")
        if self.compute_workers < 1:
            raise ValueError(f"compute_workers must be >= 1, got {self.compute_workers}")
        if self.mode == "overlapped" and self.io_agents != 1:
            raise ValueError("overlapped mode requires exactly one I/O agent")
        if self.io_agents not in (0, 1):
            raise ValueError(f"io_agents must be 0 or 1, got {self.io_agents}")
        if self.cache_budget_bytes < 0:
            raise ValueError("cache_budget_bytes must be >= 0")
        if self.prefetch_depth < 0:
            raise ValueError("prefetch_depth must be >= 0")
        if self.panel_width % 16 or not 16 <= self.panel_width <= 128:
            raise ValueError(f"panel_width must be a multiple of 16 in [16, 128], "
                             f"got {self.panel_width}")
        if self.hbm_budget_bytes < 0:
            raise ValueError("hbm_budget_bytes must be >= 0")
        if self.world_size < 0:
            raise ValueError(f"world_size must be >= 0, got {self.world_size}")
        return self

    def min_cache_tiles(self) -> int:
        return 4 * (self.prefetch_depth + 1) + 2 if self.mode == "overlapped" else 6


@dataclass
class TaskTrace:
    seq: int
    op: str
    ms_compute: float
    ms_read: float
    ms_write: float


@dataclass
class RunReport:
    """Timing / I/O accounting of one factorize or solve (task_engine.py:136-181).

    ``compute_seconds`` is device time measured with CUDA events; extra GPU
    fields: ``gpu_flops`` (algorithmic), ``gpu_tflops``, ``h2d_seconds``,
    ``d2h_seconds``.
    """

    mode: str
    task_count: int
    total_seconds: float
    compute_seconds: float
    io_read_seconds: float
    io_write_seconds: float
    tiles_read: int
    tiles_written: int
    cache_hits: int
    trace: list[TaskTrace] = field(default_factory=list, repr=False)
    gpu_flops: float = 0.0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    world_size: int = 1          # GPUs (ranks) the call ran on

    @property
    def gpu_tflops(self) -> float:
        return self.gpu_flops / self.compute_seconds / 1e12 if self.compute_seconds > 0 else 0.0

    def to_text(self) -> str:
        rows = [("mode", self.mode), ("task_count", self.task_count),
                ("total_seconds", f"{self.total_seconds:.6f}"),
                ("compute_seconds", f"{self.compute_seconds:.6f}"),
                ("io_read_seconds", f"{self.io_read_seconds:.6f}"),
                ("io_write_seconds", f"{self.io_write_seconds:.6f}"),
                ("tiles_read", self.tiles_read), ("tiles_written", self.tiles_written),
                ("cache_hits", self.cache_hits)]
        return "".join(f"{k} = {v}\n" for k, v in rows)

    def trace_csv(self) -> str:
        out = io.StringIO()
        w = csv.writer(out)
        w.writerow(["seq", "op", "ms_compute", "ms_read", "ms_write"])
        for t in self.trace:
            w.writerow([t.seq, t.op, f"{t.ms_compute:.3f}", f"{t.ms_read:.3f}",
                        f"{t.ms_write:.3f}"])
        return out.getvalue()


@dataclass
class QrFactors:
    """Persisted GPU factorization: ``factored`` (R + reflectors, reference
    layout) plus per-panel T factors and tau in raw little-endian files.

    ``device_state`` keeps the factors resident in HBM for solves in the same
    process (factor once, solve many); a fresh process re-uploads them.
    """

    factored: TiledMatrix
    inner_block: int
    rows: int
    cols: int
    tile_size: int
    panel_width: int
    geometry_hash: str = ""
    directory: Path | None = None
    device_state: QrDevice | None = field(default=None, repr=False, compare=False)
    host_state: object = field(default=None, repr=False, compare=False)  # ooc.HostStagedQR
    # (dist.DistFactors, local blocks) of this rank after a distributed factorize
    dist_state: object = field(default=None, repr=False, compare=False)

    @property
    def grid_rows(self) -> int:
        return self.factored.grid_rows

    @property
    def grid_cols(self) -> int:
        return -(-self.cols // self.tile_size)

    @property
    def s_store(self):  # reference attribute; this format keeps T in t_factors.f64
        return None

    def save_meta(self, directory) -> None:
        text = (f"rows {self.rows}\ncols {self.cols}\ntile_size {self.tile_size}\n"
                f"inner_block {self.inner_block}\ngeometry_hash {self.geometry_hash or '-'}\n"
                f"algorithm {ALGORITHM}\npanel_width {self.panel_width}\n")
        (Path(directory) / _META_NAME).write_text(text)

    @classmethod
    def load(cls, directory) -> "QrFactors":
        directory = Path(directory)
        meta = directory / _META_NAME
        if not meta.is_file():
            raise MissingFactorsError(f"no factorization at {directory}; run factorize first")
        fields = {}
        for line in meta.read_text().splitlines():
            if line.strip():
                k, v = line.split(None, 1)
                fields[k] = v.strip()
        if fields.get("algorithm") != ALGORITHM:
            raise MissingFactorsError(
                f"{directory} holds factors of algorithm {fields.get('algorithm', 'tiled-td')!r}, "
                f"not {ALGORITHM!r}")
        return cls(
            factored=TiledMatrix.open(directory / "factored"),
            inner_block=int(fields["inner_block"]), rows=int(fields["rows"]),
            cols=int(fields["cols"]), tile_size=int(fields["tile_size"]),
            panel_width=int(fields["panel_width"]),
            geometry_hash="" if fields.get("geometry_hash", "-") == "-" else fields["geometry_hash"],
            directory=directory)

    def check_complete(self) -> None:
        d = self.directory
        if d is None:
            if self.device_state is None:
                raise MissingFactorsError("factors have neither a directory nor device state")
            return
        for name in (_T_NAME, _TAU_NAME):
            if not (d / name).is_file():
                raise MissingFactorsError(f"factor file {name} missing under {d}")
        npan = -(-self.cols // self.panel_width)
        if (d / _T_NAME).stat().st_size != 8 * self.panel_width * self.panel_width * npan:
            raise MissingFactorsError(f"{d / _T_NAME} has the wrong size")
        for k in range(self.grid_cols):
            if not self.factored.tile_path(TileId(k, k)).exists():
                raise MissingFactorsError(f"factored tile ({k},{k}) missing under "
                                          f"{self.factored.directory}")

    # -- device residency -----------------------------------------------------------
    def to_device(self, device: int = 0) -> tuple[QrDevice, float, float, int]:
        """Resident QrDevice (uploading from disk if needed) + (read s, h2d s, tiles)."""
        if self.device_state is not None:
            return self.device_state, 0.0, 0.0, 0
        dev = QrDevice(self.rows, self.cols, self.panel_width, device)
        t_read = t_h2d = 0.0
        tiles = 0
        b = self.tile_size
        for j in range(self.grid_cols):
            t0 = time.perf_counter()
            try:
                blk = self.factored.read_column_block(j)
            except (OSError, CorruptTileError) as exc:
                dev.close()
                raise TaskIoError(j * self.factored.grid_rows, "load_factors", exc) from exc
            t1 = time.perf_counter()
            dev.set_matrix(blk, col0=j * b)
            t_read += t1 - t0
            t_h2d += time.perf_counter() - t1
            tiles += self.factored.grid_rows
        tau = np.fromfile(self.directory / _TAU_NAME, dtype="<f8")
        npan = -(-self.cols // self.panel_width)
        t = np.fromfile(self.directory / _T_NAME, dtype="<f8").reshape(
            (self.panel_width, npan * self.panel_width), order="F")
        dev.set_factors(tau, t)
        self.device_state = dev
        return dev, t_read, t_h2d, tiles


def _factor_dir_writes(factors: QrFactors, dev: QrDevice, directory: Path) -> tuple[float, int]:
    t0 = time.perf_counter()
    written = 0
    b = factors.tile_size
    for j in range(factors.grid_cols):
        blk = dev.get_matrix(j * b, min(b, factors.cols - j * b))
        written += factors.factored.write_column_block(j, blk)
    tau, t = dev.factors()
    tau.astype("<f8").tofile(directory / _TAU_NAME)
    t.astype("<f8").ravel(order="F").tofile(directory / _T_NAME)
    return time.perf_counter() - t0, written


def _hbm_budget(cfg: EngineConfig) -> int:
    if cfg.hbm_budget_bytes:
        return int(cfg.hbm_budget_bytes)
    import torch
    free, _ = torch.cuda.mem_get_info(cfg.device)
    return int(0.85 * free)


def _fits_in_hbm(rows: int, cols: int, cfg: EngineConfig) -> bool:
    lda = (rows + 31) // 32 * 32
    # matrix + T/R^-1 blocks + workspaces (~1 GB)
    return 8 * lda * cols + (1 << 30) <= _hbm_budget(cfg)


def _fits_in_host(rows: int, cols: int, cfg: EngineConfig) -> bool:
    lda = (rows + 31) // 32 * 32
    return 8 * lda * cols <= cfg.cache_budget_bytes


def _factorize_disk_staged(a: TiledMatrix, cfg: EngineConfig, factors_dir: Path,
                           geometry_hash: str) -> tuple["QrFactors", RunReport]:
    from .disk_ooc import DiskStagedQR
    t_start = time.perf_counter()
    b = a.tile_size
    factored = TiledMatrix.create(a.rows, a.cols, b, factors_dir / "factored")
    q = DiskStagedQR(a, factored, nb=cfg.panel_width, budget_bytes=_hbm_budget(cfg),
                     io_threads=max(1, cfg.io_agents) + 1)
    try:
        st = q.factorize()
    except (OSError, CorruptTileError) as exc:
        q.close()
        raise TaskIoError(0, "disk_staged_factorize", exc) from exc
    factors = QrFactors(factored=factored, inner_block=cfg.inner_block, rows=a.rows,
                        cols=a.cols, tile_size=b, panel_width=cfg.panel_width,
                        geometry_hash=geometry_hash, directory=factors_dir)
    q.tau.cpu().numpy()[:a.cols].astype("<f8").tofile(factors_dir / _TAU_NAME)
    q.t_all.cpu().numpy().T.astype("<f8").ravel(order="F").tofile(factors_dir / _T_NAME)
    factors.save_meta(factors_dir)
    factors.host_state = q
    report = RunReport(
        mode=cfg.mode, task_count=0, total_seconds=time.perf_counter() - t_start,
        compute_seconds=st["seconds"], io_read_seconds=st["read_s"],
        io_write_seconds=st["write_s"], tiles_read=0, tiles_written=a.grid_rows * a.grid_cols,
        cache_hits=0,
        trace=[TaskTrace(0, "qr_disk_staged_superpanels", st["seconds"] * 1e3,
                         st["read_s"] * 1e3, st["write_s"] * 1e3)],
        gpu_flops=2.0 * a.rows * a.cols ** 2 - 2.0 * a.cols ** 3 / 3.0, h2d_seconds=0.0)
    return factors, report


def _pinned_from_tiles(store: TiledMatrix, rows: int, cols: int):
    """(n, lda) pinned host tensor (column-major m x n) filled from a tile store."""
    import torch
    lda = (rows + 31) // 32 * 32
    hold = PinnedHostArray((cols, lda))      # exact size (torch's pinned allocator rounds up)
    hold.array[:] = 0.0
    host = torch.from_numpy(hold.array)
    host._qrb_pinned_hold = hold             # the registration lives as long as the tensor
    view = host.numpy().T            # lda x cols, Fortran
    b = store.tile_size
    for j in range(store.grid_cols):
        try:
            store.read_column_block(j, view[:rows, j * b:j * b + min(b, cols - j * b)])
        except (OSError, CorruptTileError) as exc:
            raise TaskIoError(j * store.grid_rows, "stage", exc) from exc
    return host


_STAGE_GBPS = 4.0       # tile read rate the left-/right-looking switch assumes (NVMe class)
_STAGE_CHUNK = 4096     # columns per gated H2D chunk (qrb_factorize_host's measured best)
_STAGE_THREADS = int(os.environ.get("QRB_IO_THREADS", "8"))  # tile readers / writers each (the
# reference has one I/O agent; positional reads and writes parallelise)


class _ColumnReader:
    """Reads the tile column blocks of ``a`` into a page-locked column-major host
    matrix on a thread pool, in column order, and raises the per-chunk ready
    flags qrb_factorize_host_gated waits on -- so the first column chunks are
    already being factored on the GPU while later tiles are still read (the
    reference overlaps I/O and compute with its one prefetching agent,
    task_engine.py:330-474).  A failed read marks every pending chunk -1 (the
    native call then returns instead of waiting) and is re-raised by join()."""

    def __init__(self, a: TiledMatrix, view: np.ndarray, chunk: int, ready: np.ndarray,
                 threads: int = _STAGE_THREADS):
        self.a, self.view, self.chunk, self.ready = a, view, chunk, ready
        self.nblk = a.grid_cols
        self.done = np.zeros(self.nblk, dtype=bool)
        self.prefix = 0                      # blocks [0, prefix) are complete
        self.lock = threading.Lock()
        self.error: BaseException | None = None
        self.error_block = 0
        self.pool = ThreadPoolExecutor(max_workers=max(1, threads))
        self.futs = []
        self.seconds = 0.0
        self.t0 = 0.0

    def _read(self, j: int) -> None:
        a, b = self.a, self.a.tile_size
        if self.error is not None:
            return
        try:
            a.read_column_block(j, self.view[:a.rows, j * b:j * b + min(b, a.cols - j * b)])
        except BaseException as exc:  # noqa: BLE001 -- re-raised in join()
            with self.lock:
                if self.error is None:
                    self.error, self.error_block = exc, j
                self.ready[self.ready == 0] = -1
            return
        with self.lock:
            self.done[j] = True
            while self.prefix < self.nblk and self.done[self.prefix]:
                self.prefix += 1
            cols = min(a.cols, self.prefix * b)
            for c in range(len(self.ready)):
                if self.ready[c] == 0 and (min(a.cols, (c + 1) * self.chunk) <= cols):
                    self.ready[c] = 1

    def start(self) -> None:
        self.t0 = time.perf_counter()
        self.futs = [self.pool.submit(self._read, j) for j in range(self.nblk)]

    def join(self) -> None:
        for f in self.futs:
            f.result()
        self.pool.shutdown(wait=True)
        self.seconds = time.perf_counter() - self.t0
        if self.error is not None:
            raise TaskIoError(self.error_block * self.a.grid_rows, "stage_a",
                              self.error) from self.error


class _ColumnWriter:
    """Streams the factored matrix into the ``factored`` tile store WHILE the
    factorization runs: a thread follows the library's progress counter
    (qrb_factorize_host_gated), copies every tile column block whose columns
    are final into a ring of page-locked buffers on its own CUDA stream, and
    hands each to a pool of positional tile writers (the reference's eager
    write-back agent, task_engine.py:330-474; written once, as there)."""

    def __init__(self, dev: QrDevice, store: TiledMatrix, progress: np.ndarray,
                 threads: int = _STAGE_THREADS):
        import torch
        self.dev, self.store, self.progress = dev, store, progress
        self.b = store.tile_size
        self.nblk = store.grid_cols
        self.lda = (store.rows + 31) // 32 * 32
        slots = max(2, threads + 2)
        self.bufs = [PinnedHostArray((self.b, self.lda)) for _ in range(slots)]
        self.busy = [None] * slots
        self.pool = ThreadPoolExecutor(max_workers=max(1, threads))
        self.stream = torch.cuda.Stream(device=dev.device)
        self.stop = False
        self.error: BaseException | None = None
        self.written = 0
        self.lock = threading.Lock()
        self.seconds = 0.0
        self.thread = threading.Thread(target=self._run, daemon=True)

    def _write(self, j: int, slot: int, w: int) -> None:
        view = self.bufs[slot].array.T[:self.store.rows, :w]      # Fortran (rows x w)
        n = self.store.write_columns(j * self.b, w, view)
        with self.lock:
            self.written += n

    def _run(self) -> None:
        t0 = time.perf_counter()
        try:
            for j in range(self.nblk):
                w = min(self.b, self.store.cols - j * self.b)
                while int(self.progress[0]) < j * self.b + w:
                    if self.stop:
                        return
                    time.sleep(0.001)
                slot = j % len(self.bufs)
                if self.busy[slot] is not None:
                    self.busy[slot].result()
                view = self.bufs[slot].array.T[:self.store.rows, :w]
                self.dev.get_matrix_async(j * self.b, w, view, self.stream.cuda_stream)
                self.stream.synchronize()
                self.busy[slot] = self.pool.submit(self._write, j, slot, w)
            for f in self.busy:
                if f is not None:
                    f.result()
        except BaseException as exc:  # noqa: BLE001 -- re-raised in join()
            self.error = exc
        finally:
            self.seconds = time.perf_counter() - t0

    def start(self) -> None:
        self.thread.start()

    def join(self, abort: bool = False) -> None:
        if abort:
            self.stop = True
        self.thread.join()
        self.pool.shutdown(wait=True)
        for buf in self.bufs:
            buf.close()
        if self.error is not None and not abort:
            raise TaskIoError(0, "write_factored", self.error) from self.error


def _factorize_host_staged(a: TiledMatrix, cfg: EngineConfig, factors_dir: Path,
                           geometry_hash: str) -> tuple["QrFactors", RunReport]:
    from .ooc import HostStagedQR
    t_start = time.perf_counter()
    t0 = time.perf_counter()
    host = _pinned_from_tiles(a, a.rows, a.cols)
    t_read = time.perf_counter() - t0
    q = HostStagedQR(host, a.rows, a.cols, nb=cfg.panel_width, budget_bytes=_hbm_budget(cfg))
    st = q.factorize()
    b = a.tile_size
    factored = TiledMatrix.create(a.rows, a.cols, b, factors_dir / "factored")
    factors = QrFactors(factored=factored, inner_block=cfg.inner_block, rows=a.rows,
                        cols=a.cols, tile_size=b, panel_width=cfg.panel_width,
                        geometry_hash=geometry_hash, directory=factors_dir)
    t1 = time.perf_counter()
    view = host.numpy().T
    written = 0
    for j in range(factored.grid_cols):
        written += factored.write_column_block(j, view[:a.rows, j * b:j * b + min(b, a.cols - j * b)])
    q.tau.cpu().numpy()[:a.cols].astype("<f8").tofile(factors_dir / _TAU_NAME)
    q.t_all.cpu().numpy().T.astype("<f8").ravel(order="F").tofile(factors_dir / _T_NAME)
    t_write = time.perf_counter() - t1
    factors.save_meta(factors_dir)
    factors.host_state = q
    report = RunReport(
        mode=cfg.mode, task_count=0, total_seconds=time.perf_counter() - t_start,
        compute_seconds=st["seconds"], io_read_seconds=t_read, io_write_seconds=t_write,
        tiles_read=a.grid_rows * a.grid_cols, tiles_written=written, cache_hits=0,
        trace=[TaskTrace(0, "stage_a_pinned", 0.0, t_read * 1e3, 0.0),
               TaskTrace(1, "qr_host_staged_superpanels", st["seconds"] * 1e3, 0.0, 0.0),
               TaskTrace(2, "write_factors", 0.0, 0.0, t_write * 1e3)],
        gpu_flops=2.0 * a.rows * a.cols ** 2 - 2.0 * a.cols ** 3 / 3.0,
        h2d_seconds=0.0)
    return factors, report


def factorize(a: TiledMatrix, config: EngineConfig, factors_dir,
              geometry_hash: str = "", keep_on_device: bool = True) -> tuple[QrFactors, RunReport]:
    """QR-factor a tiled matrix on the GPU; ``a`` itself is left untouched.

    Reference: task_engine.py:606-641.  Raises ValueError for wide matrices or
    a tile-size mismatch, TaskIoError for unreadable tiles, KernelInputError
    for non-finite entries.
    """
    if a.rows < a.cols:
        raise ValueError(f"matrix must have rows >= cols, got {a.rows}x{a.cols}")
    cfg = config.validate()
    if cfg.tile_size != a.tile_size:
        raise ValueError(f"config tile_size {cfg.tile_size} != matrix tile_size {a.tile_size}")
    factors_dir = Path(factors_dir)
    factors_dir.mkdir(parents=True, exist_ok=True)
    ctx = dist_api.context(cfg)
    if ctx is not None:                      # one process per GPU, block-cyclic columns
        return dist_api.factorize(a, cfg, factors_dir, geometry_hash, *ctx)
    if not _fits_in_hbm(a.rows, a.cols, cfg):
        if _fits_in_host(a.rows, a.cols, cfg):
            return _factorize_host_staged(a, cfg, factors_dir, geometry_hash)
        return _factorize_disk_staged(a, cfg, factors_dir, geometry_hash)
    t_start = time.perf_counter()
    dev = QrDevice(a.rows, a.cols, cfg.panel_width, cfg.device)
    b = a.tile_size
    trace: list[TaskTrace] = []
    try:
        # tiles -> page-locked column-major host matrix on reader threads, chunk
        # by chunk; the GPU copies and factors (left-looking) each chunk as soon
        # as it is complete, then finishes right-looking (qrb_factorize_host_gated)
        m, n, nb = a.rows, a.cols, cfg.panel_width
        lda = (m + 31) // 32 * 32
        chunk = max(nb, _STAGE_CHUNK // nb * nb)
        nchunks = -(-n // chunk)
        host = PinnedHostArray((n, lda))
        ready = PinnedHostArray((nchunks,), np.int32)
        ready.array[:] = 0
        view = host.array.T                                  # (lda, n), Fortran order
        reader = _ColumnReader(a, view, chunk, ready.array)
        factored = TiledMatrix.create(a.rows, a.cols, b, factors_dir / "factored")
        factors = QrFactors(factored=factored, inner_block=cfg.inner_block, rows=a.rows,
                            cols=a.cols, tile_size=b, panel_width=cfg.panel_width,
                            geometry_hash=geometry_hash, directory=factors_dir)
        progress = PinnedHostArray((1,), np.int64)
        progress.array[0] = 0
        writer = _ColumnWriter(dev, factored, progress.array)
        reader.start()
        writer.start()
        try:
            rep = dev.factorize_host_gated(view[:m], chunk, ready.array, input_gbps=_STAGE_GBPS,
                                           progress=progress.array)
        except BaseException:
            writer.join(abort=True)
            reader.join()                                    # an unreadable tile wins
            raise
        reader.join()
        t_read, t_h2d = reader.seconds, rep["h2d_ms"] / 1e3
        tiles_read = a.grid_rows * a.grid_cols
        t0 = time.perf_counter()
        writer.join()
        tau, t = dev.factors()
        tau.astype("<f8").tofile(factors_dir / _TAU_NAME)
        t.astype("<f8").ravel(order="F").tofile(factors_dir / _T_NAME)
        t_tail = time.perf_counter() - t0
        t_write, written = writer.seconds, writer.written
        host.close()
        ready.close()
        progress.close()
        trace.append(TaskTrace(0, "stage_a_overlapped", 0.0, t_read * 1e3, 0.0))
        trace.append(TaskTrace(1, "qr_geqrf_cwy", rep["total_ms"], 0.0, 0.0))
        trace.append(TaskTrace(2, "write_factors_overlapped", 0.0, 0.0, t_write * 1e3))
        trace.append(TaskTrace(3, "write_tail_after_qr", 0.0, 0.0, t_tail * 1e3))
        factors.save_meta(factors_dir)
    except BaseException:
        dev.close()
        raise
    if keep_on_device:
        factors.device_state = dev
    else:
        dev.close()
    report = RunReport(
        mode=cfg.mode, task_count=int(rep["kernel_launches"]),
        total_seconds=time.perf_counter() - t_start, compute_seconds=rep["total_ms"] / 1e3,
        io_read_seconds=t_read, io_write_seconds=t_write, tiles_read=tiles_read,
        tiles_written=written, cache_hits=0, trace=trace, gpu_flops=rep["flops"],
        h2d_seconds=t_h2d)
    return factors, report


def solve(factors: QrFactors, b_mat: TiledMatrix, config: EngineConfig,
          out_dir) -> tuple[TiledMatrix, RunReport]:
    """Least-squares X = R^-1 (Q^T B) for every column of ``b_mat`` on the GPU.

    Reference: task_engine.py:644-685 (same checks and errors; B untouched;
    X written to ``out_dir/x``).  A zero / sub-1e-300 pivot raises
    SingularMatrixError naming the column the reference would name.
    """
    cfg = config.validate()
    if b_mat.rows != factors.rows:
        raise ValueError(f"right-hand side has {b_mat.rows} rows, factors expect {factors.rows}")
    if b_mat.tile_size != factors.tile_size:
        raise ValueError(f"right-hand side tile_size {b_mat.tile_size} != factors "
                         f"tile_size {factors.tile_size}")
    if cfg.inner_block != factors.inner_block:
        raise ValueError(f"config inner_block {cfg.inner_block} != factorization inner_block "
                         f"{factors.inner_block}; applies must reuse the factorization width")
    factors.check_complete()
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    ctx = dist_api.context(cfg)
    if ctx is not None:                      # slices split over the ranks
        return dist_api.solve(factors, b_mat, cfg, out_dir, *ctx)
    if factors.host_state is not None or (factors.device_state is None and
                                          not _fits_in_hbm(factors.rows, factors.cols, cfg)):
        return _solve_host_staged(factors, b_mat, cfg, out_dir)
    t_start = time.perf_counter()
    dev, t_read_f, t_h2d_f, tiles_f = factors.to_device(cfg.device)
    b = b_mat.tile_size
    t0 = time.perf_counter()
    try:
        bm = np.empty((b_mat.rows, b_mat.cols), order="F")
        for j in range(b_mat.grid_cols):
            b_mat.read_column_block(j, bm[:, j * b:j * b + min(b, b_mat.cols - j * b)])
    except (OSError, CorruptTileError, CacheCapacityError) as exc:
        raise TaskIoError(0, "stage_b", exc) from exc
    t_read = time.perf_counter() - t0 + t_read_f
    x, _resid, rep = dev.solve(bm, report_block=factors.tile_size)
    t1 = time.perf_counter()
    xm = TiledMatrix.create(factors.cols, b_mat.cols, b, out_dir / "x")
    written = 0
    for j in range(xm.grid_cols):
        written += xm.write_column_block(j, x[:, j * b:j * b + min(b, b_mat.cols - j * b)])
    t_write = time.perf_counter() - t1
    trace = [TaskTrace(0, "stage_b", 0.0, t_read * 1e3, 0.0),
             TaskTrace(1, "ormqr_trsm", rep["total_ms"], 0.0, 0.0),
             TaskTrace(2, "write_x", 0.0, 0.0, t_write * 1e3)]
    report = RunReport(
        mode=cfg.mode, task_count=int(rep["kernel_launches"]),
        total_seconds=time.perf_counter() - t_start, compute_seconds=rep["total_ms"] / 1e3,
        io_read_seconds=t_read, io_write_seconds=t_write,
        tiles_read=tiles_f + b_mat.grid_rows * b_mat.grid_cols, tiles_written=written,
        cache_hits=0, trace=trace, gpu_flops=rep["flops"],
        h2d_seconds=t_h2d_f + rep["h2d_ms"] / 1e3, d2h_seconds=rep["d2h_ms"] / 1e3)
    return xm, report


def _solve_host_staged(factors: "QrFactors", b_mat: TiledMatrix, cfg: EngineConfig,
                       out_dir: Path) -> tuple[TiledMatrix, RunReport]:
    import torch

    from .disk_ooc import DiskStagedQR
    from .ooc import HostStagedQR
    t_start = time.perf_counter()
    q = factors.host_state
    if q is None and not _fits_in_host(factors.rows, factors.cols, cfg):
        q = DiskStagedQR(None, factors.factored, nb=factors.panel_width,
                         budget_bytes=_hbm_budget(cfg))
        npan = -(-factors.cols // factors.panel_width)
        nb = factors.panel_width
        tau = np.fromfile(factors.directory / _TAU_NAME, dtype="<f8")
        t = np.fromfile(factors.directory / _T_NAME, dtype="<f8").reshape((nb, npan * nb),
                                                                          order="F")
        q.tau[:factors.cols] = torch.from_numpy(tau).cuda()
        q.t_all.copy_(torch.from_numpy(np.ascontiguousarray(t.T)).cuda())
        factors.host_state = q
    if q is None:
        host = _pinned_from_tiles(factors.factored, factors.rows, factors.cols)
        q = HostStagedQR(host, factors.rows, factors.cols, nb=factors.panel_width,
                         budget_bytes=_hbm_budget(cfg))
        npan = -(-factors.cols // factors.panel_width)
        nb = factors.panel_width
        tau = np.fromfile(factors.directory / _TAU_NAME, dtype="<f8")
        t = np.fromfile(factors.directory / _T_NAME, dtype="<f8").reshape((nb, npan * nb),
                                                                          order="F")
        q.tau[:factors.cols] = torch.from_numpy(tau).cuda()
        q.t_all.copy_(torch.from_numpy(np.ascontiguousarray(t.T)).cuda())
        factors.host_state = q
    lda = q.lda
    bm = np.empty((b_mat.rows, b_mat.cols), order="F")
    b = b_mat.tile_size
    try:
        for j in range(b_mat.grid_cols):
            b_mat.read_column_block(j, bm[:, j * b:j * b + min(b, b_mat.cols - j * b)])
    except (OSError, CorruptTileError, CacheCapacityError) as exc:
        raise TaskIoError(0, "stage_b", exc) from exc
    b_dev = torch.zeros((b_mat.cols, lda), dtype=torch.float64, device="cuda")
    b_dev[:, :b_mat.rows] = torch.from_numpy(np.ascontiguousarray(bm.T)).cuda()
    t0 = time.perf_counter()
    x, _ = q.solve(b_dev, report_block=factors.tile_size)
    t_compute = time.perf_counter() - t0
    x = x.cpu().numpy().T
    xm = TiledMatrix.create(factors.cols, b_mat.cols, b, out_dir / "x")
    written = 0
    for j in range(xm.grid_cols):
        written += xm.write_column_block(j, x[:, j * b:j * b + min(b, b_mat.cols - j * b)])
    report = RunReport(
        mode=cfg.mode, task_count=0, total_seconds=time.perf_counter() - t_start,
        compute_seconds=t_compute, io_read_seconds=0.0, io_write_seconds=0.0,
        tiles_read=b_mat.grid_rows * b_mat.grid_cols, tiles_written=written, cache_hits=0,
        trace=[TaskTrace(0, "host_staged_solve", t_compute * 1e3, 0.0, 0.0)],
        gpu_flops=(4.0 * factors.rows * factors.cols - factors.cols ** 2) * b_mat.cols)
    return xm, report


__all__ = ["EngineConfig", "RunReport", "TaskTrace", "QrFactors", "factorize", "solve",
           "SingularMatrixError"]
