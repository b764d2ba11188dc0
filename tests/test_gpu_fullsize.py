"""Parity at BASELINE.json's full sizes (configs 2 and 3), where the CPU oracle
is infeasible: cross-checks against cuSOLVER (torch fp64) at
config 2 and size-independent properties at config 3 (residual identity, the
Gram identity R^T R = A^T A on sampled columns, norm preservation of Q^T,
run-to-run bitwise determinism)."""

import numpy as np
import pytest

from paper_1907_01891_b200 import ct_system as cs

pytestmark = pytest.mark.gpu


def _setup(cfg, slices):
    import torch
    from paper_1907_01891_b200.device import QrDevice
    g = cs.config_geometry(cfg)
    m, n = g.n_rays, g.n_pixels
    lda = (m + 31) // 32 * 32
    a = cs.densify_device(g, lda)
    x_true = cs.phantom_stack_device(cfg, slices)
    b = torch.zeros((slices, lda), dtype=torch.float64, device="cuda")
    b[:, :m] = x_true @ a[:, :m]
    q = QrDevice(m, n)
    q.set_matrix_device(a)
    q.factorize()
    x = torch.zeros((slices, n), dtype=torch.float64, device="cuda")
    r = torch.zeros(slices, dtype=torch.float64, device="cuda")
    q.solve_device(b, x, r)
    return g, a, b, q, x, r, x_true


def test_config2_against_cusolver():
    import torch
    g, a, b, q, x, r, x_true = _setup(2, 8)
    m, n = g.n_rays, g.n_pixels
    A = a[:, :m].T                                   # m x n (strided view)
    R_ref = torch.linalg.qr(A.contiguous(), mode="r")[1]
    R = torch.from_numpy(q.r_factor()).cuda()
    s = torch.sign(torch.diagonal(R)) * torch.sign(torch.diagonal(R_ref))
    err_r = float((R * s[:, None] - R_ref).abs().max() / R_ref.abs().max())
    assert err_r <= 1e-10, err_r
    x_ref = torch.linalg.lstsq(A.contiguous(), b[:, :m].T.contiguous()).solution.T
    err_x = float((x - x_ref).abs().max() / x_ref.abs().max())
    assert err_x <= 1e-8, err_x
    # noiseless sinograms: the solution is the phantom itself
    assert float((x - x_true).abs().max() / x_true.abs().max()) <= 1e-8
    res = torch.linalg.norm(x @ a[:, :m] - b[:, :m], dim=1)
    assert float(((res - r).abs() / torch.clamp(res, min=1e-300)).max()) <= 1e-6 or \
        float(res.max()) <= 1e-9 * float(b.abs().max())
    q.close()


def test_config3_size_independent_properties():
    import torch
    g, a, b, q, x, r, x_true = _setup(3, 4)
    m, n = g.n_rays, g.n_pixels
    # noiseless b = A x_true: the QR solve recovers the phantom
    assert float((x - x_true).abs().max() / x_true.abs().max()) <= 1e-8
    # residual identity ||(Q^T b)[n:m]|| = ||A x - b|| (both ~0 here) and small
    res = torch.linalg.norm(x @ a[:, :m] - b[:, :m], dim=1)
    bn = torch.linalg.norm(b[:, :m], dim=1)
    assert float((res / bn).max()) <= 1e-12 and float((r / bn).max()) <= 1e-12
    # Gram identity on sampled columns: (R^T R)[:, j] = A^T a_j
    rng = np.random.default_rng(3)
    cols = np.sort(rng.choice(n, 16, replace=False))
    fact = torch.from_numpy(q.get_matrix(0, n)).cuda()          # m x n
    R = torch.triu(fact[:n])
    lhs = R.T @ R[:, cols]
    rhs = a[:, :m] @ a[cols, :m].T
    assert float((lhs - rhs).abs().max() / rhs.abs().max()) <= 1e-10
    del fact, R
    # run-to-run bitwise determinism of the whole factorization + solve
    x1 = x.clone()
    q.set_matrix_device(a)
    q.factorize()
    x2 = torch.zeros_like(x)
    q.solve_device(b, x2, torch.zeros_like(r))
    assert torch.equal(x1, x2)
    q.close()


def test_config2_against_reference_golden():
    """BASELINE config 2 against the REFERENCE package itself
    (tests/golden/make_golden_cfg2.py: oocqr factorize + solve on the same
    Siddon matrix, tile 2048, inner block 128): X <= 1e-8, residual <= 1e-9,
    |diag R| and the first rows of R (row signs normalised) <= 1e-10."""
    import hashlib
    from pathlib import Path

    import torch
    from paper_1907_01891_b200.device import QrDevice
    fx = Path(__file__).resolve().parent / "golden" / "ref_ct2.npz"
    if not fx.is_file():
        pytest.skip("config-2 reference fixture not generated")
    ref = np.load(fx)
    g = cs.config_geometry(2)
    m, n = g.n_rays, g.n_pixels
    assert str(ref["geometry_hash"]) == cs.geometry_hash(g)
    lda = (m + 31) // 32 * 32
    a = cs.densify_device(g, lda)
    a_host = np.ascontiguousarray(a[:, :m].cpu().numpy().T)          # same bytes, C order
    assert hashlib.sha256(a_host.tobytes()).hexdigest() == str(ref["a_sha256"])
    del a_host
    bm = ref["b"]
    b = torch.zeros((bm.shape[1], lda), dtype=torch.float64, device="cuda")
    b[:, :m] = torch.from_numpy(np.ascontiguousarray(bm.T)).cuda()
    q = QrDevice(m, n)
    q.set_matrix_device(a)
    q.factorize()
    x = torch.zeros((bm.shape[1], n), dtype=torch.float64, device="cuda")
    r = torch.zeros(bm.shape[1], dtype=torch.float64, device="cuda")
    q.solve_device(b, x, r)
    xr = ref["x"]
    assert np.abs(x.cpu().numpy().T - xr).max() <= 1e-8 * np.abs(xr).max()
    np.testing.assert_allclose(r.cpu().numpy(), ref["resid"], rtol=1e-9)
    rd = np.abs(q.rdiag())
    assert np.abs(rd - ref["rdiag_abs"]).max() <= 1e-10 * ref["rdiag_abs"].max()
    rows = q.get_matrix(0, n)[:4]                                     # 4 x n
    rows = np.array([np.where(np.arange(n) >= i, rows[i], 0.0) for i in range(4)])
    rows = rows * np.sign(np.diag(rows[:, :4]))[:, None]
    assert np.abs(rows - ref["r_rows4"]).max() <= 1e-10 * np.abs(ref["r_rows4"]).max()
    q.close()


@pytest.mark.parametrize("cfg,fixture", [(6, "ref_ct4r.npz"), (8, "ref_ct4q.npz")])
def test_reduced_config4_family_against_reference_golden(cfg, fixture):
    """Config 4's geometry family at 1/8 width (4230 x 4096) and 1/4 width
    (16920 x 16384), m/n = 1.03 as at full size: the GPU factorization + solve
    against the reference package's own result (tests/golden/make_golden_cfg4r.py,
    make_golden_cfg4q.py) -- the parity pin for config 4, whose 566 GB the
    reference cannot factor here."""
    from pathlib import Path

    import torch
    from paper_1907_01891_b200.device import QrDevice
    ref = np.load(Path(__file__).resolve().parent / "golden" / fixture)
    g = cs.config_geometry(cfg)
    m, n = g.n_rays, g.n_pixels
    lda = (m + 31) // 32 * 32
    a = cs.densify_device(g, lda)
    bm = ref["b"]
    b = torch.zeros((bm.shape[1], lda), dtype=torch.float64, device="cuda")
    b[:, :m] = torch.from_numpy(np.ascontiguousarray(bm.T)).cuda()
    q = QrDevice(m, n)
    q.set_matrix_device(a)
    q.factorize()
    x = torch.zeros((bm.shape[1], n), dtype=torch.float64, device="cuda")
    r = torch.zeros(bm.shape[1], dtype=torch.float64, device="cuda")
    q.solve_device(b, x, r)
    xr = ref["x"]
    assert np.abs(x.cpu().numpy().T - xr).max() <= 1e-8 * np.abs(xr).max()
    np.testing.assert_allclose(r.cpu().numpy(), ref["resid"], rtol=1e-9)
    assert np.abs(np.abs(q.rdiag()) - ref["rdiag_abs"]).max() <= 1e-10 * ref["rdiag_abs"].max()
    rows = q.get_matrix(0, n)[:8]
    rows = np.array([np.where(np.arange(n) >= i, rows[i], 0.0) for i in range(8)])
    rows = rows * np.sign(np.diag(rows[:, :8]))[:, None]
    assert np.abs(rows - ref["r_rows8"]).max() <= 1e-10 * np.abs(ref["r_rows8"]).max()
    q.close()
