"""The multi-GPU driver's CUDA path, exercised as a single NCCL rank on one
GPU (the distributed schedule itself is covered over gloo in test_dist_cpu)."""

import os
import socket

import numpy as np
import pytest

from conftest import rel_err, sign_normalise
from oracle import tiled_qr as orc

pytestmark = pytest.mark.gpu


def test_single_rank_nccl_factor_gather_solve():
    import torch
    import torch.distributed as dist
    from paper_1907_01891_b200 import dist as qd
    from paper_1907_01891_b200.device import QrDevice

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(11)
        m, n, nb = 700, 333, 64
        a = rng.standard_normal((m, n))
        lda = (m + 31) // 32 * 32
        full = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
        full[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
        a_local = qd.scatter_block_cyclic(full, n, nb, 0, 1)
        f = qd.factorize_distributed(a_local, m, n, nb, lda, 0, 1, qd.CudaOps())
        fact = f.a_local[:, :m].cpu().numpy().T
        ref = orc.factorize_dense(a, 128, 64)
        assert rel_err(sign_normalise(np.triu(fact[:n])), sign_normalise(ref.r())) <= 1e-10
        q = QrDevice(m, n, nb)
        qd.gather_factored(f, place=lambda k, panel: q.set_matrix_device(panel, col0=k * nb))
        q.set_factors(f.tau_all.cpu().numpy()[:n], f.t_all.cpu().numpy().T.copy(order="F"))
        np.testing.assert_array_equal(q.get_matrix(), fact)
        bm = rng.standard_normal((m, 5))
        x, _, _ = q.solve(bm)
        assert rel_err(x, orc.solve_dense(ref, bm)) <= 1e-8
        q.close()
        # panel-pair blocks: the factors gathered in place under a view handle, the
        # broadcast pair reflectors handed to the solve (no second merge, no copy)
        bw = 2 * nb
        a2 = qd.scatter_block_cyclic(full, n, bw, 0, 1)
        f2 = qd.factorize_distributed(a2, m, n, nb, lda, 0, 1, qd.CudaOps(), bw=bw)
        assert f2.t2_blocks is not None
        store = qd.gather_storage(n, bw, 1, lda, a2.device)
        qd.gather_into(f2, store)
        qv = QrDevice.view(store, m, n, nb)
        qv.set_factors(f2.tau_all.cpu().numpy()[:n], f2.t_all.cpu().numpy().T.copy(order="F"))
        from paper_1907_01891_b200 import _native
        old_min = _native.get_tuning("t4_min_rhs")
        _native.set_tuning("t4_min_rhs", 0)               # merge pairs / quads at the solve
        try:
            x_lazy, _, _ = qv.solve(bm)                   # pairs merged by the solve
            qv.set_factors(f2.tau_all.cpu().numpy()[:n],
                           f2.t_all.cpu().numpy().T.copy(order="F"))
            qv.set_pair_factors(f2.t2_blocks)
            x_given, _, _ = qv.solve(bm)                  # pairs as broadcast
        finally:
            _native.set_tuning("t4_min_rhs", old_min)
        np.testing.assert_array_equal(x_given, x_lazy)
        assert rel_err(x_given, orc.solve_dense(ref, bm)) <= 1e-8
        qv.close()
        # memory-lean solve straight from the distributed factors
        bsh = torch.zeros((5, lda), dtype=torch.float64, device="cuda")
        bsh[:, :m] = torch.from_numpy(np.ascontiguousarray(bm.T)).cuda()
        x2, r2 = qd.solve_distributed(f, bsh, qd.CudaOps())
        assert rel_err(x2.cpu().numpy().T, orc.solve_dense(ref, bm)) <= 1e-8
        np.testing.assert_allclose(r2.cpu().numpy(), orc.residual_norms(ref, bm), rtol=1e-9)
    finally:
        dist.destroy_process_group()


def _bench_line(cmd, root):
    import json
    import subprocess
    res = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    return json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("launcher", ["torchrun", "self"])
def test_bench_multirank_path_two_ranks_gloo(tmp_path, launcher):
    """bench.py's multi-GPU path (dist.bench_rank: per-rank Siddon densify,
    all-reduced sinograms, block-cyclic factorization with the owner's side-
    stream look-ahead, gather, slice-split solve, e2e) end to end with 2 ranks
    -- under torchrun, and as `python bench.py --gpus 2` with no launcher (the
    script starts its ranks itself) -- here over gloo with both ranks on the one
    GPU, so the control flow of an N = 2 run is exercised (not its
    performance; the line says so: "ranks" 2, "n_gpus" = GPUs actually used)."""
    import sys
    from pathlib import Path

    import torch
    root = Path(__file__).resolve().parent.parent
    args = ["--gpus", "2", "--config", "2", "--dist-backend", "gloo", "--steps", "1",
            "--warmup", "1"]
    if launcher == "torchrun":
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
               "2", "--master-addr", "127.0.0.1", "--master-port", str(port),
               str(root / "bench.py"), *args]
    else:
        cmd = [sys.executable, str(root / "bench.py"), *args]
    line = _bench_line(cmd, root)
    assert line["ranks"] == 2 and line["n_gpus"] == min(2, torch.cuda.device_count())
    assert line["backend"] == "gloo" and "FUNCTIONAL CHECK" in line["config"]["parallelism"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["slices_per_s"] > 0 and line["gpu_launches"] > 0
