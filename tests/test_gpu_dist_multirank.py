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
