"""Multi-GPU behind the drop-in ``factorize`` / ``solve`` (reference
task_engine.py:606-685): one process per GPU, SPMD.

Every rank of an initialized ``torch.distributed`` process group (NCCL, one
GPU per rank; launched e.g. with ``torchrun --nproc-per-node 8``) calls the
reference's ``factorize(a, config, factors_dir)`` / ``solve(factors, b,
config, out_dir)`` with the same arguments.  With ``EngineConfig.world_size``
0 (auto: the process group's size) or equal to it, the call is routed here:

factorize
  * each rank stages only its own column blocks (1D block-cyclic, width
    bw = 2 nb: block k lives on rank k % G) from the tile store -- one scatter
    ``preadv`` per (tile, column range), tile_store.read_columns -- into pinned
    memory and HBM;
  * ``dist.factorize_distributed``: per block the owner factors it and
    broadcasts (V, T2, tau) over NCCL; the owner of the next block factors it
    on a side stream under its own capped trailing update (look-ahead);
  * each rank writes its factored columns straight into their tiles of
    ``factors_dir/factored`` (disjoint column ranges of the same tile files:
    ``pwritev``, no locking needed); rank 0 writes T, tau and ``meta.txt``.
    The directory is the single-GPU format, so a later single-GPU (or
    differently sized) run can solve from it.

solve
  * the singularity rule of the reference (bottom-up tiles of ``tile_size``,
    first |R_jj| < 1e-300 or NaN, kernels.py:423-426 / task_engine.py:246-253)
    is applied to the GLOBAL diagonal of R (each rank contributes its blocks'
    entries, one all-reduce) before any work, so every rank raises the same
    ``SingularMatrixError`` the reference would;
  * slices (columns of B) are split evenly; a rank reads only its share of B;
  * if a replica of the factors fits next to the local blocks, the factored
    panels are all-gathered into one ``QrDevice`` per rank and each rank solves
    its share with no further communication; otherwise (config 4: 566 GB) the
    memory-lean solve streams V and R by per-panel broadcasts;
  * each rank writes its X columns into ``out_dir/x``.

The reference has no distributed code.  ``_ops`` / ``_device``
exist for the gloo CPU tests (numpy local arithmetic); the product path always
uses the CUDA library (dist.CudaOps) and fails if it is missing.
"""

from __future__ import annotations

import os
import time
from pathlib import Path

import numpy as np

from . import dist as qd
from .errors import CorruptTileError, KernelInputError, TaskIoError
from .tile_store import TiledMatrix


def context(cfg):
    """(rank, world) when the call must run distributed, else None."""
    try:
        import torch.distributed as dist
        ready = dist.is_available() and dist.is_initialized()
    except ImportError:  # pragma: no cover
        ready = False
    if not ready:
        if cfg.world_size > 1:
            raise ValueError(f"EngineConfig.world_size={cfg.world_size} needs an initialized "
                             f"torch.distributed process group (one process per GPU)")
        return None
    world = dist.get_world_size()
    if cfg.world_size == 1 or world == 1:
        return None
    if cfg.world_size not in (0, world):
        raise ValueError(f"EngineConfig.world_size={cfg.world_size} but the process group has "
                         f"{world} ranks")
    return dist.get_rank(), world


def _device(cfg):
    import torch
    if not torch.cuda.is_available():
        from .errors import NativeUnavailableError
        raise NativeUnavailableError("distributed factorize/solve needs one CUDA GPU per rank")
    local = int(os.environ.get("LOCAL_RANK", cfg.device))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    return torch.device("cuda", dev)


def local_blocks(n: int, bw: int, rank: int, world: int) -> list[tuple[int, int, int]]:
    """(global block k, first column, width) of this rank's blocks, local order."""
    nblk = -(-n // bw)
    return [(k, k * bw, min(bw, n - k * bw)) for k in qd.local_panels(nblk, rank, world)]


def read_local_blocks(store: TiledMatrix, blocks, bw: int, host_cm: np.ndarray) -> int:
    """Columns of this rank's blocks from the tile files into ``host_cm``
    (Fortran view, ld >= rows, local block i at columns [i bw, i bw + w))."""
    reads = 0
    for i, (_, c0, w) in enumerate(blocks):
        reads += store.read_columns(c0, w, 0, host_cm[:, i * bw:i * bw + w])
    return reads


def write_local_blocks(store: TiledMatrix, blocks, bw: int, host_cm: np.ndarray) -> int:
    """This rank's factored columns into their tiles (disjoint column ranges)."""
    writes = 0
    for i, (_, c0, w) in enumerate(blocks):
        writes += store.write_columns(c0, w, host_cm[:store.rows, i * bw:i * bw + w])
    return writes


def _max_over_ranks(x: float, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def factorize(a: TiledMatrix, cfg, factors_dir: Path, geometry_hash: str, rank: int, world: int,
              _ops=None, _device_override=None):
    """The distributed drop-in factorization (module docstring)."""
    import torch
    import torch.distributed as dist

    from .task_engine import QrFactors, RunReport, TaskTrace, _T_NAME, _TAU_NAME
    t_start = time.perf_counter()
    dev = _device_override or _device(cfg)
    ops = _ops or qd.CudaOps(world)
    m, n, nb = a.rows, a.cols, cfg.panel_width
    bw = 2 * nb
    lda = (m + 31) // 32 * 32
    blocks = local_blocks(n, bw, rank, world)
    n_local = sum(w for _, _, w in blocks)
    pin = dev.type == "cuda"
    host = torch.zeros((max(n_local, 1), lda), dtype=torch.float64, pin_memory=pin)
    view = host.numpy().T                                   # lda x n_local, Fortran
    t0 = time.perf_counter()
    err = None
    try:
        tiles_read = read_local_blocks(a, blocks, bw, view)
    except (OSError, CorruptTileError) as exc:
        err, tiles_read = exc, 0
    t_read = time.perf_counter() - t0
    flag = torch.tensor([1.0 if err else 0.0], dtype=torch.float64, device=dev)
    dist.all_reduce(flag)                                  # every rank raises together
    if float(flag):
        raise TaskIoError(0, "stage_a", err or OSError("tile read failed on another rank"))
    a_local = host[:n_local].to(dev, non_blocking=True) if n_local else \
        torch.zeros((0, lda), dtype=torch.float64, device=dev)
    bad = torch.tensor([0.0 if bool(torch.isfinite(a_local).all()) else 1.0],
                       dtype=torch.float64, device=dev)
    dist.all_reduce(bad)
    if float(bad):
        raise KernelInputError("factorize: input matrix has non-finite entries")
    f = qd.factorize_distributed(a_local, m, n, nb, lda, rank, world, ops, bw=bw)
    compute_s = _max_over_ranks(f.factor_seconds, dev)
    # factored columns -> their tiles; rank 0 creates the store first
    t1 = time.perf_counter()
    if rank == 0:
        TiledMatrix.create(m, n, a.tile_size, factors_dir / "factored")
    dist.barrier()
    factored = TiledMatrix.open(factors_dir / "factored")
    host[:n_local].copy_(f.a_local)
    written = write_local_blocks(factored, blocks, bw, view)
    if rank == 0:
        f.tau_all.cpu().numpy()[:n].astype("<f8").tofile(factors_dir / _TAU_NAME)
        f.t_all.cpu().numpy().astype("<f8").ravel().tofile(factors_dir / _T_NAME)
    factors = QrFactors(factored=factored, inner_block=cfg.inner_block, rows=m, cols=n,
                        tile_size=a.tile_size, panel_width=nb, geometry_hash=geometry_hash,
                        directory=factors_dir)
    if rank == 0:
        factors.save_meta(factors_dir)
    dist.barrier()
    t_write = time.perf_counter() - t1
    factors.dist_state = (f, blocks)
    report = RunReport(
        mode=cfg.mode, task_count=0, total_seconds=time.perf_counter() - t_start,
        compute_seconds=compute_s, io_read_seconds=t_read, io_write_seconds=t_write,
        tiles_read=tiles_read, tiles_written=written, cache_hits=0,
        trace=[TaskTrace(0, f"stage_local_blocks_rank{rank}", 0.0, t_read * 1e3, 0.0),
               TaskTrace(1, f"qr_block_cyclic_{world}ranks", compute_s * 1e3, 0.0, 0.0),
               TaskTrace(2, "write_local_blocks", 0.0, 0.0, t_write * 1e3)],
        gpu_flops=2.0 * m * n ** 2 - 2.0 * n ** 3 / 3.0, world_size=world)
    return factors, report


def _load_local(factors, cfg, rank, world, dev):
    """DistFactors of this rank from a factors directory (a later process)."""
    import torch
    nb = factors.panel_width
    bw = 2 * nb
    m, n = factors.rows, factors.cols
    lda = (m + 31) // 32 * 32
    blocks = local_blocks(n, bw, rank, world)
    n_local = sum(w for _, _, w in blocks)
    host = torch.zeros((max(n_local, 1), lda), dtype=torch.float64, pin_memory=dev.type == "cuda")
    try:
        read_local_blocks(factors.factored, blocks, bw, host.numpy().T)
        tau = np.fromfile(factors.directory / "tau.f64", dtype="<f8")
        npan = -(-n // nb)
        t = np.fromfile(factors.directory / "t_factors.f64", dtype="<f8").reshape(npan * nb, nb)
    except (OSError, CorruptTileError, ValueError) as exc:
        raise TaskIoError(0, "load_factors", exc) from exc
    a_local = host[:n_local].to(dev)
    f = qd.DistFactors(m, n, nb, lda, rank, world, a_local,
                       torch.from_numpy(np.ascontiguousarray(t)).to(dev),
                       torch.from_numpy(tau).to(dev), 0.0, {}, bw)
    return f, blocks


def solve(factors, b_mat: TiledMatrix, cfg, out_dir: Path, rank: int, world: int,
          _ops=None, _device_override=None, _replicate: bool | None = None):
    """The distributed drop-in solve (module docstring)."""
    import torch
    import torch.distributed as dist

    from .task_engine import RunReport, TaskTrace
    t_start = time.perf_counter()
    dev = _device_override or _device(cfg)
    ops = _ops or qd.CudaOps(world)
    state = getattr(factors, "dist_state", None)
    if state is not None and state[0].world == world:
        f, blocks = state
    else:
        f, blocks = _load_local(factors, cfg, rank, world, dev)
        factors.dist_state = (f, blocks)
    m, n, lda = f.m, f.n, f.lda
    qd.check_singular(f, factors.tile_size)       # before any work, on every rank
    S = b_mat.cols
    first, cnt = qd.slice_share(S, rank, world)
    host = torch.zeros((max(cnt, 1), lda), dtype=torch.float64, pin_memory=dev.type == "cuda")
    t0 = time.perf_counter()
    err = None
    try:
        if cnt:
            b_mat.read_columns(first, cnt, 0, host.numpy().T)
    except (OSError, CorruptTileError) as exc:
        err = exc
    flag = torch.tensor([1.0 if err else 0.0], dtype=torch.float64, device=dev)
    dist.all_reduce(flag)
    if float(flag):
        raise TaskIoError(0, "stage_b", err or OSError("tile read failed on another rank"))
    t_read = time.perf_counter() - t0
    b_dev = host.to(dev)
    if _replicate is None:
        free = torch.cuda.mem_get_info(dev)[0] if dev.type == "cuda" else 0
        _replicate = dev.type == "cuda" and 8 * lda * n * 1.1 < 0.8 * free
    t1 = time.perf_counter()
    if _replicate:
        from .device import QrDevice
        store = qd.gather_storage(n, f.block, f.world, f.lda, dev)
        qd.gather_into(f, store)
        q = QrDevice.view(store, m, n, f.nb, dev.index or 0)
        try:
            q.set_factors(f.tau_all.cpu().numpy()[:n], f.t_all.cpu().numpy().T.copy(order="F"))
            if f.t2_blocks is not None:
                q.set_pair_factors(f.t2_blocks)
            x = torch.zeros((max(cnt, 1), n + (n & 1)), dtype=torch.float64, device=dev)
            if cnt:
                q.solve_device(b_dev[:cnt], x[:cnt], report_block=factors.tile_size)
            x = x[:cnt, :n]
        finally:
            q.close()
        path = "all-gathered factors, per-rank solve"
    else:
        x, _ = qd.solve_distributed(f, b_dev[:cnt], ops, report_block=factors.tile_size)
        path = "memory-lean: V and R streamed by per-panel broadcasts"
    ops.sync()
    compute_s = _max_over_ranks(time.perf_counter() - t1, dev)
    t2 = time.perf_counter()
    if rank == 0:
        TiledMatrix.create(n, S, b_mat.tile_size, out_dir / "x")
    dist.barrier()
    xm = TiledMatrix.open(out_dir / "x")
    written = 0
    if cnt:
        xh = np.asfortranarray(x.cpu().numpy().T)
        written = xm.write_columns(first, cnt, xh)
    dist.barrier()
    t_write = time.perf_counter() - t2
    report = RunReport(
        mode=cfg.mode, task_count=0, total_seconds=time.perf_counter() - t_start,
        compute_seconds=compute_s, io_read_seconds=t_read, io_write_seconds=t_write,
        tiles_read=0, tiles_written=written, cache_hits=0,
        trace=[TaskTrace(0, f"stage_b_share_rank{rank}", 0.0, t_read * 1e3, 0.0),
               TaskTrace(1, f"solve_{world}ranks ({path})", compute_s * 1e3, 0.0, 0.0),
               TaskTrace(2, "write_x_share", 0.0, 0.0, t_write * 1e3)],
        gpu_flops=(4.0 * m * n - n * n) * S, world_size=world)
    return xm, report
