"""The distributed drop-in (dist_api: every rank calls the reference's
factorize / solve on the same tile stores) as 2 and 3 CPU processes over gloo,
with the test-only numpy local arithmetic of test_dist_cpu.  Checks the host
logic the GPU path shares: block-cyclic staging from the tile files, the
factored store written by all ranks into the same tiles, the T / tau files,
the slice split of B and X, and the reference's singular-column order."""

import os
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tiled_qr as orc
from paper_1907_01891_b200 import dist as qd
from paper_1907_01891_b200 import dist_api
from paper_1907_01891_b200.errors import SingularMatrixError
from paper_1907_01891_b200.task_engine import EngineConfig, QrFactors
from paper_1907_01891_b200.tile_store import TiledMatrix, gather_matrix, scatter_matrix
from test_dist_cpu import NumpyOps, free_port


def _matrix(m, n, zero_cols=()):
    rng = np.random.default_rng(17)
    a = rng.standard_normal((m, n))
    for c in zero_cols:
        a[:, c] = 0.0
    return a, rng.standard_normal((m, 5))


def _worker(rank, world, port, m, n, b, nb, root, zero_cols):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = EngineConfig(tile_size=b, inner_block=min(nb, b), panel_width=nb).validate()
        assert dist_api.context(cfg) == (rank, world)
        a_store = TiledMatrix.open(os.path.join(root, "a"))
        b_store = TiledMatrix.open(os.path.join(root, "b"))
        cpu = torch.device("cpu")
        factors, rep = dist_api.factorize(a_store, cfg, Path(root, "f"),
                                          "geo", rank, world, _ops=NumpyOps(),
                                          _device_override=cpu)
        assert rep.world_size == world
        try:
            dist_api.solve(factors, b_store, cfg, Path(root, "out"), rank,
                           world, _ops=NumpyOps(), _device_override=cpu, _replicate=False)
        except SingularMatrixError as exc:
            with open(os.path.join(root, f"singular_{rank}.txt"), "w") as fh:
                fh.write(str(exc.global_column))
        # a later "process": solve from the directory alone (no dist_state)
        f2 = QrFactors.load(os.path.join(root, "f"))
        try:
            dist_api.solve(f2, b_store, cfg, Path(root, "out2"), rank,
                           world, _ops=NumpyOps(), _device_override=cpu, _replicate=False)
        except SingularMatrixError as exc:
            with open(os.path.join(root, f"singular2_{rank}.txt"), "w") as fh:
                fh.write(str(exc.global_column))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,b,nb", [(2, 300, 200, 64, 32), (3, 257, 250, 96, 16),
                                            (2, 130, 128, 128, 16)])
def test_distributed_dropin_matches_oracle(tmp_path, world, m, n, b, nb):
    a, bm = _matrix(m, n)
    scatter_matrix(TiledMatrix.create(m, n, b, tmp_path / "a"), a)
    scatter_matrix(TiledMatrix.create(m, bm.shape[1], b, tmp_path / "b"), bm)
    mp.spawn(_worker, args=(world, free_port(), m, n, b, nb, str(tmp_path), ()), nprocs=world,
             join=True)
    f = orc.factorize_dense(a, 64, 32)
    fact = gather_matrix(TiledMatrix.open(tmp_path / "f" / "factored"))
    r = np.triu(fact[:n])
    r_ref = f.r()
    s = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
    assert np.abs(r * s[:, None] - r_ref).max() <= 1e-10 * np.abs(r_ref).max()
    x_ref = orc.solve_dense(f, bm)
    for out in ("out", "out2"):
        x = gather_matrix(TiledMatrix.open(tmp_path / out / "x"))
        assert x.shape == (n, bm.shape[1])
        assert np.abs(x - x_ref).max() <= 1e-8 * np.abs(x_ref).max()
    # T / tau / meta written once, in the single-GPU format
    meta = QrFactors.load(tmp_path / "f")
    assert (meta.rows, meta.cols, meta.panel_width, meta.geometry_hash) == (m, n, nb, "geo")
    meta.check_complete()
    assert np.fromfile(tmp_path / "f" / "tau.f64").size == n


@pytest.mark.parametrize("zero_cols,expect", [((6,), 6), ((3, 19), 19), ((0,), 0)])
def test_distributed_singular_column_order(tmp_path, zero_cols, expect):
    """Exactly-zero columns: every rank raises the column the reference's
    bottom-up tile order names (tile 8: {3, 19} -> 19), whatever the block
    (2 nb = 32) and rank layout."""
    m, n, b, nb = 40, 24, 8, 16
    a, bm = _matrix(m, n, zero_cols)
    scatter_matrix(TiledMatrix.create(m, n, b, tmp_path / "a"), a)
    scatter_matrix(TiledMatrix.create(m, bm.shape[1], b, tmp_path / "b"), bm)
    mp.spawn(_worker, args=(2, free_port(), m, n, b, nb, str(tmp_path), zero_cols), nprocs=2,
             join=True)
    for rank in range(2):
        for name in ("singular", "singular2"):
            assert int((tmp_path / f"{name}_{rank}.txt").read_text()) == expect


def test_context_rules():
    assert dist_api.context(EngineConfig(world_size=0)) is None       # no process group
    assert dist_api.context(EngineConfig(world_size=1)) is None
    with pytest.raises(ValueError):
        dist_api.context(EngineConfig(world_size=2))
    with pytest.raises(ValueError):
        EngineConfig(world_size=-1).validate()


def test_singular_column_rule_matches_reference_order():
    d = np.ones(24)
    d[[3, 19]] = 0.0
    assert qd.singular_column(d, 8) == 19
    d = np.ones(24)
    d[[9, 14]] = [np.nan, 0.0]
    assert qd.singular_column(d, 8) == 9
    assert qd.singular_column(np.ones(5), 8) == -1
    d = np.ones(24)
    d[2] = 1e-301
    assert qd.singular_column(d, 0) == 2
