"""Host-staged (out-of-HBM) factorization and solve vs the oracle."""

import numpy as np
import pytest

from conftest import rel_err, sign_normalise
from oracle import tiled_qr as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,sp_pairs,nb", [(3000, 2000, 2, 128), (1500, 1500, 1, 64),
                                               (2500, 700, 3, 32), (2600, 2330, 3, 128)])
def test_host_staged_matches_oracle(m, n, sp_pairs, nb):
    import torch
    from paper_1907_01891_b200.ooc import HostStagedQR

    rng = np.random.default_rng(m + n)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.linspace(50, 1, n)) @ v.T
    lda = (m + 31) // 32 * 32
    a_host = torch.zeros((n, lda), dtype=torch.float64, pin_memory=True)
    a_host[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T))
    col_bytes = 8 * lda
    # budget: the super-panel (a whole number of panel pairs) + two pair-wide V buffers
    q = HostStagedQR(a_host, m, n, nb=nb, budget_bytes=(2 * sp_pairs + 4) * col_bytes * nb)
    assert q.sp_cols == min(n, sp_pairs * 2 * nb)
    st = q.factorize()
    assert st["super_panels"] == -(-n // q.sp_cols)
    f = orc.factorize_dense(a, 256, 64)
    r = np.triu(a_host[:, :n].numpy().T)
    assert rel_err(sign_normalise(r), sign_normalise(f.r())) <= 1e-10
    bm = rng.standard_normal((m, 6))
    b_dev = torch.zeros((6, lda), dtype=torch.float64, device="cuda")
    b_dev[:, :m] = torch.from_numpy(np.ascontiguousarray(bm.T)).cuda()
    x, resid = q.solve(b_dev)
    x_ref = orc.solve_dense(f, bm)
    assert rel_err(x.cpu().numpy().T, x_ref) <= 1e-8
    np.testing.assert_allclose(resid.cpu().numpy(), orc.residual_norms(f, bm), rtol=1e-9,
                               atol=1e-12 * np.linalg.norm(bm, axis=0).max())


def test_dropin_api_switches_to_host_staging(tmp_path):
    """factorize/solve with an HBM budget smaller than A take the host-staged path
    and still match the oracle (and a later process can solve from disk)."""
    import paper_1907_01891_b200 as pkg
    rng = np.random.default_rng(5)
    m, n, b = 1200, 900, 128
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.linspace(20, 1, n)) @ v.T
    bm = rng.standard_normal((m, 4))
    am = pkg.TiledMatrix.create(m, n, b, tmp_path / "a")
    pkg.scatter_matrix(am, a)
    rhs = pkg.TiledMatrix.create(m, 4, b, tmp_path / "b")
    pkg.scatter_matrix(rhs, bm)
    lda = (m + 31) // 32 * 32
    cfg = pkg.EngineConfig(tile_size=b, inner_block=64,
                           hbm_budget_bytes=8 * lda * 300 + (1 << 30) - 1)   # < A + 1 GB
    factors, rep = pkg.factorize(a=am, config=cfg, factors_dir=tmp_path / "f")
    assert factors.host_state is not None and rep.trace[1].op == "qr_host_staged_superpanels"
    f = orc.factorize_dense(a, 256, 64)
    r = np.triu(pkg.gather_matrix(factors.factored)[:n, :n])
    assert rel_err(sign_normalise(r), sign_normalise(f.r())) <= 1e-10
    x, _ = pkg.solve(factors, rhs, cfg, tmp_path / "out")
    assert rel_err(pkg.gather_matrix(x), orc.solve_dense(f, bm)) <= 1e-8
    loaded = pkg.QrFactors.load(tmp_path / "f")
    x2, _ = pkg.solve(loaded, rhs, cfg, tmp_path / "out2")
    assert rel_err(pkg.gather_matrix(x2), orc.solve_dense(f, bm)) <= 1e-8
