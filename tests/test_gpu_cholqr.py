"""CholeskyQR2 + Householder-reconstruction panel (csrc/cholqr.cu) against the
column-by-column Householder panel (the reference's dlarfg recurrence,
kernels.py:74-131) and against the oracle.

The reconstruction chooses each reflector sign on the fly exactly as dlarfg
does, so the factors are not just "R up to row sign": R, V, tau and T agree
with the Householder panel to rounding (checked here at 1e-10 relative)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


@pytest.fixture(params=[63, 7, 0], ids=["warp_diag4", "warp_diag", "barrier_diag"])
def native(request):
    """Every test of this module runs with the 128 x 128 factorizations'
    diagonal steps shared by four warps (Cholesky, LU; the default), all in one
    warp, and as the 8-warp barrier versions
    (qrb tuning "sf_diag", csrc/smallfact.cu)."""
    from paper_1907_01891_b200 import _native
    lib = _native.load()
    algo, rows = _native.get_tuning("panel_algo"), _native.get_tuning("cholqr_min_rows")
    diag = _native.get_tuning("sf_diag")
    _native.set_tuning("sf_diag", request.param)
    yield _native, lib
    _native.set_tuning("panel_algo", algo)
    _native.set_tuning("cholqr_min_rows", rows)
    _native.set_tuning("sf_diag", diag)


def _panel(lib, a_np, algo, native_mod):
    """Factor the m x w panel a_np with the given algorithm; returns (P, tau, T)."""
    m, w = a_np.shape
    ld = m + (m & 1)
    a = torch.zeros((w, ld), dtype=torch.float64, device="cuda")
    a[:, :m] = torch.from_numpy(np.ascontiguousarray(a_np.T)).cuda()
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    t = torch.zeros((w, w), dtype=torch.float64, device="cuda")
    native_mod.set_tuning("panel_algo", algo)
    native_mod.check(lib.qrb_op_panel(_p(a), ld, m, w, _p(tau), _p(t), w, None), "qrb_op_panel")
    torch.cuda.synchronize()
    return a[:, :m].cpu().numpy().T, tau.cpu().numpy(), t.cpu().numpy().T


@pytest.mark.parametrize("m,w", [(256, 128), (2160, 128), (5000, 96), (17280, 128), (69120, 128)])
def test_cholqr2_panel_matches_householder_panel(native, m, w):
    nat, lib = native
    rng = np.random.default_rng(m + w)
    a = rng.standard_normal((m, w))
    before = (nat.get_tuning("cholqr_panels"), nat.get_tuning("cholqr_fallbacks"))
    p2, tau2, t2 = _panel(lib, a, 2, nat)
    after = (nat.get_tuning("cholqr_panels"), nat.get_tuning("cholqr_fallbacks"))
    assert after[0] == before[0] + 1 and after[1] == before[1], "CholeskyQR2 route not taken"
    p1, tau1, t1 = _panel(lib, a, 1, nat)
    r1, r2 = np.triu(p1[:w]), np.triu(p2[:w])
    assert np.abs(r2 - r1).max() <= 1e-10 * np.abs(r1).max()
    v1, v2 = np.tril(p1, -1), np.tril(p2, -1)
    assert np.abs(v2 - v1).max() <= 1e-10 * max(1.0, np.abs(v1).max())
    assert np.abs(tau2 - tau1).max() <= 1e-12
    assert np.abs(np.triu(t2) - np.triu(t1)).max() <= 1e-10 * np.abs(t1).max()
    # factors reproduce A: Q R with Q = I - V T V^T applied to [R; 0]
    v = np.tril(p2, -1) + np.eye(m, w)
    qr_ = np.vstack([r2, np.zeros((m - w, w))])
    qr_ = qr_ - v @ (np.triu(t2) @ (v.T @ qr_))
    assert np.linalg.norm(qr_ - a) <= 1e-12 * np.linalg.norm(a) * np.sqrt(m)


def test_cholqr2_falls_back_on_rank_deficient_panel(native):
    nat, lib = native
    rng = np.random.default_rng(7)
    a = rng.standard_normal((6000, 128))
    a[:, 17] = 0.0                       # reference convention: sigma = 0 -> tau = 0
    a[:, 40] = a[:, 3]                   # dependent column
    f0 = nat.get_tuning("cholqr_fallbacks")
    p2, tau2, t2 = _panel(lib, a, 2, nat)
    assert nat.get_tuning("cholqr_fallbacks") == f0 + 1
    p1, tau1, t1 = _panel(lib, a, 1, nat)
    np.testing.assert_array_equal(p2, p1)
    np.testing.assert_array_equal(tau2, tau1)
    assert tau2[17] == 0.0


def test_cholqr2_falls_back_on_ill_conditioned_panel(native):
    nat, lib = native
    rng = np.random.default_rng(8)
    u, _ = np.linalg.qr(rng.standard_normal((8000, 128)))
    v, _ = np.linalg.qr(rng.standard_normal((128, 128)))
    a = (u * np.logspace(0, -11, 128)) @ v.T        # cond 1e11 > 1/sqrt(eps)
    f0 = nat.get_tuning("cholqr_fallbacks")
    _panel(lib, a, 2, nat)
    assert nat.get_tuning("cholqr_fallbacks") == f0 + 1


@pytest.mark.parametrize("algo", [0, 2])
def test_factorize_and_solve_with_cholqr2_panels(native, algo):
    """Whole QR + solve with the CholeskyQR2 panel against the oracle restatement."""
    nat, _ = native
    from oracle.tiled_qr import factorize_dense
    from paper_1907_01891_b200.device import QrDevice
    from conftest import sign_normalise

    nat.set_tuning("panel_algo", algo)
    nat.set_tuning("cholqr_min_rows", 1024)
    m, n = 3000, 768
    rng = np.random.default_rng(11)
    a = rng.standard_normal((m, n))
    b = rng.standard_normal((m, 5))
    p0 = nat.get_tuning("cholqr_panels")
    with QrDevice(m, n) as q:
        q.set_matrix(a)
        q.factorize()
        r_gpu = q.r_factor()
        x_gpu, res_gpu, _ = q.solve(b)
    assert nat.get_tuning("cholqr_panels") - p0 == n // 128
    r_ref = np.triu(factorize_dense(a, 256, 128).r())
    assert np.abs(sign_normalise(r_gpu) - sign_normalise(r_ref)).max() <= 1e-10 * np.abs(r_ref).max()
    x_ref = np.linalg.lstsq(a, b, rcond=None)[0]
    assert np.abs(x_gpu - x_ref).max() <= 1e-8 * np.abs(x_ref).max()
    res_ref = np.linalg.norm(a @ x_ref - b, axis=0)
    np.testing.assert_allclose(res_gpu, res_ref, rtol=1e-9)


def test_cholqr2_moderately_conditioned_panel_takes_the_full_second_pass(native):
    """cond ~1e5: ||Q1^T Q1 - I|| ~ 1e-6 is above the closed-form threshold, so
    the second Cholesky runs as a full sweep -- still the Householder factors."""
    nat, lib = native
    rng = np.random.default_rng(21)
    m, w = 9000, 128
    u, _ = np.linalg.qr(rng.standard_normal((m, w)))
    v, _ = np.linalg.qr(rng.standard_normal((w, w)))
    a = (u * np.logspace(0, -5, w)) @ v.T
    f0 = nat.get_tuning("cholqr_fallbacks")
    p2, tau2, t2 = _panel(lib, a, 2, nat)
    assert nat.get_tuning("cholqr_fallbacks") == f0
    p1, tau1, t1 = _panel(lib, a, 1, nat)
    r1, r2 = np.triu(p1[:w]), np.triu(p2[:w])
    assert np.abs(r2 - r1).max() <= 1e-9 * np.abs(r1).max()
    assert np.abs(tau2 - tau1).max() <= 1e-9
    v2 = np.tril(p2, -1) + np.eye(m, w)
    q = np.eye(m) - v2 @ np.triu(t2) @ v2.T
    assert np.linalg.norm(q.T @ q - np.eye(m)) <= 1e-12
