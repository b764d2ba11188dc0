"""The multi-GPU schedule (1D block-cyclic panels, one broadcast per panel,
slice-split solve) run as 2 and 3 CPU processes over gloo with numpy local
arithmetic; the result must equal the single-process oracle factorization."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tiled_qr as orc
from paper_1907_01891_b200 import dist as qd


def unit_lower(p):
    v = np.tril(p, -1)
    d = min(p.shape)
    v[np.arange(d), np.arange(d)] = 1.0
    return v


def strided(t, off, rows, cols, ld):
    flat = t.numpy().reshape(-1)
    return np.lib.stride_tricks.as_strided(flat[off:], shape=(rows, cols), strides=(8, ld * 8))


class NumpyOps:
    """Test-only local arithmetic: the oracle's Householder sweep (kernels.py:80-101)
    and T recurrence (kernels.py:134-147) on an m x w panel."""

    def panel(self, a, lda, row0, col0, m, w, tau, t, ldt):
        p = strided(a, row0 + col0 * lda, m, w, lda)
        taus = orc._factor_columns(lambda c: (p[c], p[c + 1:]), 0, w)
        v = unit_lower(p)
        tf = orc._t_factor(lambda k: v[:, :k].T @ v[:, k], taus)
        tau.numpy()[:w] = taus
        strided(t, 0, w, w, ldt)[:, :] = tf

    def panel_block(self, a, lda, row0, col0, m, w, nb, tau, t2, ldt2, side=False):
        """w <= 2 nb columns as one Householder sweep: the compact-WY T of the
        whole block equals the merged pair reflector the GPU op builds."""
        self.panel(a, lda, row0, col0, m, w, tau, t2, ldt2)

    def apply_qt(self, v, ldv, v_off, m, w, t, ldt, c, ldc, c_off, nc):
        if nc <= 0:
            return
        vu = unit_lower(strided(v, v_off, m, w, ldv).copy())
        tf = strided(t, 0, w, w, ldt).copy()
        cm = strided(c, c_off, m, nc, ldc)
        cm -= vu @ (tf.T @ (vu.T @ cm))

    def trsm_upper(self, r, ldr, r_off, n, b, ldb, b_off, nrhs):
        rm = np.triu(strided(r, r_off, n, n, ldr).copy())
        bm = strided(b, b_off, n, nrhs, ldb)
        bm[:, :] = np.linalg.solve(rm, bm)

    def gemm_nn_sub(self, a, lda, a_off, m, k, bmat, ldb, b_off, c, c_off, n):
        am = strided(a, a_off, m, k, lda).copy()
        bm = strided(bmat, b_off, k, n, ldb).copy()
        cm = strided(c, c_off, m, n, ldb)
        cm -= am @ bm

    def sync(self):
        pass


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def worker(rank, world, port, m, n, nb, out_dir, lookahead=True, bw=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    a = rng.standard_normal((m, n))
    lda = m + (m & 1)
    full = torch.zeros((n, lda), dtype=torch.float64)
    full[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T))
    bw = bw or nb
    a_local = qd.scatter_block_cyclic(full, n, bw, rank, world)
    assert a_local.shape[0] == qd.local_cols(n, bw, rank, world)
    f = qd.factorize_distributed(a_local, m, n, nb, lda, rank, world, NumpyOps(),
                                 lookahead=lookahead, bw=bw)
    fact = qd.gather_factored(f)
    # the in-place round-wise gather (global column order, no reorder copy)
    store = qd.gather_storage(n, f.block, world, lda, a_local.device)
    qd.gather_into(f, store)
    assert torch.equal(store[:n], fact), "gather_into differs from gather_factored"
    if rank == 0:
        np.save(os.path.join(out_dir, "factored.npy"), fact[:, :m].numpy().T)
        np.save(os.path.join(out_dir, "t_all.npy"), f.t_all.numpy())
    # slice-split solve: every rank solves its share against the gathered factors
    bmat = rng.standard_normal((m, 7))
    first, cnt = qd.slice_share(7, rank, world)
    fm = fact[:, :m].numpy().T.copy()
    c = bmat[:, first:first + cnt].copy()
    for k in range(-(-n // nb)):
        j0, pw = k * nb, min(nb, n - k * nb)
        vu = unit_lower(fm[j0:, j0:j0 + pw])
        tf = f.t_all.numpy()[k * nb:k * nb + pw, :pw].T
        c[j0:] -= vu @ (tf.T @ (vu.T @ c[j0:]))
    x = np.linalg.solve(np.triu(fm[:n, :n]), c[:n])
    np.save(os.path.join(out_dir, f"x_{rank}.npy"), x)
    # memory-lean solve: panels and R block columns broadcast, no gather
    bsh = torch.zeros((cnt, lda), dtype=torch.float64)
    bsh[:, :m] = torch.from_numpy(np.ascontiguousarray(bmat[:, first:first + cnt].T))
    x2, r2 = qd.solve_distributed(f, bsh, NumpyOps())
    np.save(os.path.join(out_dir, f"x2_{rank}.npy"), x2.numpy().T)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,nb,la,bw", [(2, 300, 200, 32, True, 32),
                                                (3, 257, 250, 16, True, 16),
                                                (2, 64, 40, 16, True, 16),
                                                (2, 300, 200, 32, False, 32),
                                                (4, 200, 150, 16, True, 16),
                                                (2, 300, 200, 32, True, 64),
                                                (3, 257, 250, 16, True, 32),
                                                (2, 300, 200, 32, False, 64)])
def test_block_cyclic_factorization_matches_oracle(tmp_path, world, m, n, nb, la, bw):
    mp.spawn(worker, args=(world, free_port(), m, n, nb, str(tmp_path), la, bw), nprocs=world,
             join=True)
    rng = np.random.default_rng(7)
    a = rng.standard_normal((m, n))
    fact = np.load(tmp_path / "factored.npy")
    f = orc.factorize_dense(a, 64, 32)
    r_ref = f.r()
    r = np.triu(fact[:n])
    s = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
    assert np.abs(r * s[:, None] - r_ref).max() <= 1e-10 * np.abs(r_ref).max()
    bmat = rng.standard_normal((m, 7))
    x_ref = orc.solve_dense(f, bmat)
    parts = []
    for r_ in range(world):
        first, cnt = qd.slice_share(7, r_, world)
        parts.append(np.load(tmp_path / f"x_{r_}.npy"))
        assert parts[-1].shape == (n, cnt)
    x = np.concatenate(parts, axis=1)
    assert np.abs(x - x_ref).max() <= 1e-8 * np.abs(x_ref).max()
    x2 = np.concatenate([np.load(tmp_path / f"x2_{r_}.npy") for r_ in range(world)], axis=1)
    assert np.abs(x2 - x_ref).max() <= 1e-8 * np.abs(x_ref).max()


def test_ownership_helpers():
    # panel pairs (bw = 2 nb): panel 5 is the second panel of block 2 -> rank 0 at local col 32+16
    assert qd.panel_home(5, 16, 32, 2) == (0, 48)
    assert qd.panel_home(2, 16, 32, 2) == (1, 0)
    assert qd.local_panels(10, 1, 4) == [1, 5, 9]
    assert qd.first_local_after(5, 1, 4) == 2   # panels 1, 5 done -> next local is 9
    assert qd.first_local_after(0, 3, 4) == 0
    assert sum(qd.local_cols(1000, 128, r, 3) for r in range(3)) == 1000
    shares = [qd.slice_share(4096, r, 8) for r in range(8)]
    assert shares[0] == (0, 512) and sum(c for _, c in shares) == 4096


def test_config4_memory_plan_at_8_gpus():
    """BASELINE config 4 (270000 x 262144 fp64, 566 GB) on 8 x B200 (180 GB):
    ~71 GB of A per rank, two ~553 MB block-broadcast buffers, and no room for
    a replica of the factors, so the solve is the memory-lean streamed one;
    config 3 (36 GB) replicates."""
    hbm = 179e9
    p = qd.memory_plan(270000, 262144, 128, 8, hbm)
    assert p["local_cols"] == 32768
    assert abs(p["local_bytes"] - 70.8e9) < 0.1e9
    assert p["bcast_buffers"] == 2 and abs(p["bcast_buffer_bytes"] - 553.5e6) < 1e6
    assert p["fits"] and p["lean_solve"] and p["total_bytes"] < 75e9
    p3 = qd.memory_plan(69120, 65536, 128, 8, hbm)
    assert not p3["lean_solve"] and p3["fits"]
    # one GPU cannot hold config 4 at all (the host-staged tier takes over)
    assert not qd.memory_plan(270000, 262144, 128, 1, hbm)["fits"]


def test_owner_chain_sms_grows_when_the_update_is_short():
    """The owner's SM split (dist.owner_chain_sms): the look-ahead's 24 SMs while
    its capped update hides the block chain, more SMs in the late steps where
    the chain is the critical path of every rank."""
    from paper_1907_01891_b200.dist import owner_chain_sms
    # config 3 at 8 GPUs, first step: 8192 local trailing columns, m = 69120
    assert owner_chain_sms(69120, 8192, 256, 68864, 128) == 24
    # late step: 1024 local columns left, m_k = 6000 -> chain-bound
    late = owner_chain_sms(6000, 1024, 256, 5744, 128)
    assert late > 24
    # monotone in the remaining update
    assert owner_chain_sms(20000, 512, 256, 19744, 128) >= owner_chain_sms(20000, 4096, 256,
                                                                           19744, 128)
