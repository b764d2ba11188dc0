"""The multi-GPU driver with its CUDA local arithmetic (CudaOps: the sm_100a
kernels) and 2-3 ranks, all on the one GPU this harness has, exchanging panels
over gloo.  gloo moves the data through host memory, so no rank's kernel ever
waits on another rank's kernel (the ranks' contexts are simply time-sliced):
this is a functional check of the block-cyclic schedule, the look-ahead
broadcast buffers, the gather and the memory-lean solve on real device
buffers -- not a stand-in for multi-GPU performance."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, n, nb, out_dir, lookahead, bw, side, h2d=False):
    import torch.distributed as dist

    from paper_1907_01891_b200 import dist as qd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        a = rng.standard_normal((m, n))
        lda = (m + 31) // 32 * 32
        full = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
        full[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
        a_local = qd.scatter_block_cyclic(full, n, bw, rank, world)
        ops = qd.CudaOps(world, side_lookahead=side)
        host = None
        if h2d:  # local blocks streamed in from pinned host memory during the first steps
            host = a_local.cpu().pin_memory()
            a_local.zero_()
        f = qd.factorize_distributed(a_local, m, n, nb, lda, rank, world, ops,
                                     lookahead=lookahead, bw=bw, host_src=host, chunk_cols=192)
        fact = qd.gather_factored(f)
        bmat = rng.standard_normal((m, 6))
        first, cnt = qd.slice_share(6, rank, world)
        bsh = torch.zeros((max(cnt, 1), lda), dtype=torch.float64, device="cuda")
        bsh[:cnt, :m] = torch.from_numpy(np.ascontiguousarray(bmat[:, first:first + cnt].T)).cuda()
        x2, r2 = qd.solve_distributed(f, bsh[:cnt], ops)
        np.save(os.path.join(out_dir, f"x2_{rank}.npy"), x2.cpu().numpy().T)
        np.save(os.path.join(out_dir, f"r2_{rank}.npy"), r2.cpu().numpy())
        if rank == 0:
            np.save(os.path.join(out_dir, "factored.npy"), fact[:, :m].cpu().numpy().T)
            np.save(os.path.join(out_dir, "b.npy"), bmat)
            np.save(os.path.join(out_dir, "a.npy"), a)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,nb,la,bw,side", [(2, 1500, 700, 128, True, 128, False),
                                                     (3, 1100, 900, 64, True, 64, False),
                                                     (2, 900, 500, 32, False, 32, False),
                                                     (2, 1500, 700, 64, True, 128, True),
                                                     (3, 1100, 900, 64, True, 128, True),
                                                     (1, 1500, 1000, 64, True, 128, True),
                                                     (2, 900, 500, 32, False, 64, True),
                                                     (2, 1500, 1000, 64, True, 128, "h2d"),
                                                     (1, 1500, 1000, 64, True, 128, "h2d")])
def test_multirank_cuda_schedule_matches_oracle(tmp_path, world, m, n, nb, la, bw, side):
    """bw = 2 nb: panel-pair blocks (qrb_op_panel_block); side: the owner's next
    block factored + broadcast on a side stream under its capped update; "h2d":
    the local blocks copied in from pinned host memory by chunks during the
    first steps (host_src)."""
    import torch.multiprocessing as mp

    from conftest import rel_err, sign_normalise
    from oracle import tiled_qr as orc

    mp.spawn(_worker, args=(world, _free_port(), m, n, nb, str(tmp_path), la, bw, bool(side),
                            side == "h2d"), nprocs=world, join=True)
    a = np.load(tmp_path / "a.npy")
    bmat = np.load(tmp_path / "b.npy")
    fact = np.load(tmp_path / "factored.npy")
    ref = orc.factorize_dense(a, 256, 64)
    assert rel_err(sign_normalise(np.triu(fact[:n])), sign_normalise(ref.r())) <= 1e-10
    x_ref = orc.solve_dense(ref, bmat)
    r_ref = orc.residual_norms(ref, bmat)
    for rank in range(world):
        from paper_1907_01891_b200 import dist as qd
        first, cnt = qd.slice_share(6, rank, world)
        if cnt == 0:
            continue
        x2 = np.load(tmp_path / f"x2_{rank}.npy")
        assert rel_err(x2, x_ref[:, first:first + cnt]) <= 1e-8
        np.testing.assert_allclose(np.load(tmp_path / f"r2_{rank}.npy"), r_ref[first:first + cnt],
                                   rtol=1e-9)


def _dropin_worker(rank, world, port, root, m, n, b, nb):
    import torch.distributed as dist

    import paper_1907_01891_b200 as pkg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = pkg.EngineConfig(tile_size=b, inner_block=128, panel_width=nb)   # world_size 0: auto
        a = pkg.TiledMatrix.open(os.path.join(root, "a"))
        bm = pkg.TiledMatrix.open(os.path.join(root, "b"))
        factors, rep = pkg.factorize(a, cfg, os.path.join(root, "f"))
        assert rep.world_size == world and factors.dist_state is not None
        pkg.solve(factors, bm, cfg, os.path.join(root, "out"))
        # a later process: solve from the directory (each rank re-reads its blocks)
        f2 = pkg.QrFactors.load(os.path.join(root, "f"))
        pkg.solve(f2, bm, cfg, os.path.join(root, "out2"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,b,nb", [(2, 1500, 1100, 512, 64), (3, 900, 700, 256, 32)])
def test_dropin_factorize_solve_routes_to_block_cyclic_ranks(tmp_path, world, m, n, b, nb):
    """The reference API itself (factorize / solve) called by every rank of a
    process group: routed to dist_api (block-cyclic factorization with the CUDA
    kernels, slice-split solve, every rank writing its own columns of the
    stores); the result is the single-process oracle's."""
    import torch.multiprocessing as mp

    import paper_1907_01891_b200 as pkg
    from oracle import tiled_qr as orc
    rng = np.random.default_rng(23)
    a = rng.standard_normal((m, n))
    bmat = rng.standard_normal((m, 5))
    pkg.scatter_matrix(pkg.TiledMatrix.create(m, n, b, tmp_path / "a"), a)
    pkg.scatter_matrix(pkg.TiledMatrix.create(m, 5, b, tmp_path / "b"), bmat)
    mp.spawn(_dropin_worker, args=(world, _free_port(), str(tmp_path), m, n, b, nb),
             nprocs=world, join=True)
    f = orc.factorize_dense(a, 128, 32)
    fact = pkg.gather_matrix(pkg.TiledMatrix.open(tmp_path / "f" / "factored"))
    r, r_ref = np.triu(fact[:n]), f.r()
    s = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
    assert np.abs(r * s[:, None] - r_ref).max() <= 1e-10 * np.abs(r_ref).max()
    x_ref = orc.solve_dense(f, bmat)
    for out in ("out", "out2"):
        x = pkg.gather_matrix(pkg.TiledMatrix.open(tmp_path / out / "x"))
        assert np.abs(x - x_ref).max() <= 1e-8 * np.abs(x_ref).max()
    # the factors directory is the single-GPU format: one process solves from it too
    x1 = pkg.solve(pkg.QrFactors.load(tmp_path / "f"), pkg.TiledMatrix.open(tmp_path / "b"),
                   pkg.EngineConfig(tile_size=b, panel_width=nb, world_size=1), tmp_path / "o1")[0]
    assert np.abs(pkg.gather_matrix(x1) - x_ref).max() <= 1e-8 * np.abs(x_ref).max()
