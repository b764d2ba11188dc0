"""Kernel-level parity of the stream-ordered C-ABI operators (qrb_op_*)."""

import ctypes

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import rel_err
from oracle import tiled_qr as orc
from paper_1907_01891_b200 import _native

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def lib():
    return _native.load()


def to_dev(a, ld=None):
    """numpy (rows x cols) -> torch (cols, ld) holding the column-major matrix."""
    a = np.asarray(a, dtype=np.float64)
    ld = ld or a.shape[0] + (a.shape[0] & 1)
    t = torch.zeros((a.shape[1], ld), dtype=torch.float64, device="cuda")
    t[:, :a.shape[0]] = torch.from_numpy(np.ascontiguousarray(a.T))
    return t, ld


def to_host(t, rows):
    torch.cuda.synchronize()
    return t[:, :rows].cpu().numpy().T.copy()


def P(t, off=0):
    return ctypes.c_void_p(t.data_ptr() + 8 * off)


def unit_lower(v):
    d = min(v.shape)
    u = np.tril(v, -1)
    u[np.arange(d), np.arange(d)] = 1.0
    return u


@pytest.mark.parametrize("m,n,k", [(128, 64, 16), (300, 70, 37), (1000, 513, 128), (64, 8, 3),
                                   (4616, 5, 128), (130, 1, 1)])
def test_gemm_nn_sub(m, n, k):
    rng = np.random.default_rng(m + n + k)
    A, B, C = (rng.standard_normal(s) for s in [(m, k), (k, n), (m, n)])
    At, lda = to_dev(A)
    Bt, ldb = to_dev(B)
    Ct, ldc = to_dev(C)
    assert lib().qrb_op_gemm_nn_sub(P(At), lda, P(Bt), ldb, P(Ct), ldc, m, n, k, None) == 0
    assert rel_err(to_host(Ct, m), C - A @ B) <= 1e-13


@pytest.mark.parametrize("m,n,k", [(2160, 256, 128), (2032, 896, 128), (1000, 130, 256), (300, 70, 37)])
def test_gemm_nn_sub_few_tiles_128x32_is_bitwise_the_128x64_result(m, n, k):
    """Updates with few 128 x 64 tiles run 128 x 32 tiles (qrb tuning
    "few_tiles_bn32", csrc/gemm_dmma.cu): same K order per element and C - acc
    rounded once either way, so the two kernels agree bit for bit."""
    from paper_1907_01891_b200 import _native
    rng = np.random.default_rng(m * 7 + n + k)
    A, B, C = (rng.standard_normal(s) for s in [(m, k), (k, n), (m, n)])
    At, lda = to_dev(A)
    Bt, ldb = to_dev(B)
    keep = _native.get_tuning("few_tiles_bn32")
    out = []
    try:
        for knob in (0, 2):
            _native.set_tuning("few_tiles_bn32", knob)
            Ct, ldc = to_dev(C)
            assert lib().qrb_op_gemm_nn_sub(P(At), lda, P(Bt), ldb, P(Ct), ldc, m, n, k, None) == 0
            out.append(to_host(Ct, m))
    finally:
        _native.set_tuning("few_tiles_bn32", keep)
    np.testing.assert_array_equal(out[0], out[1])
    assert rel_err(out[1], C - A @ B) <= 1e-13


@pytest.mark.parametrize("k,m,n,splits", [(4616, 128, 5, 1), (4616, 128, 5, 18), (5000, 40, 70, 3),
                                          (48, 128, 128, 4), (1000, 128, 1000, 2), (17, 3, 2, 1)])
@pytest.mark.parametrize("mask_a,mask_b", [(0, 0), (1, 0), (1, 1)])
def test_gemm_tn_with_unit_lower_masks(k, m, n, splits, mask_a, mask_b):
    rng = np.random.default_rng(k + m + n)
    A, B = rng.standard_normal((k, m)), rng.standard_normal((k, n))
    Ae = unit_lower(A) if mask_a else A
    Be = unit_lower(B) if mask_b else B
    At, lda = to_dev(A)
    Bt, ldb = to_dev(B)
    Ct, ldc = to_dev(np.zeros((m, n)))
    st = lib().qrb_op_gemm_tn(P(At), lda, P(Bt), ldb, P(Ct), ldc, m, n, k, splits, mask_a, mask_b,
                              None)
    assert st == 0
    assert rel_err(to_host(Ct, m), Ae.T @ Be) <= 1e-13


@pytest.mark.parametrize("m,w", [(64, 64), (500, 128), (2160, 128), (20000, 128), (70000, 128),
                                 (3000, 56), (129, 1), (4000, 100)])
def test_panel_matches_lapack_geqrf(m, w):
    rng = np.random.default_rng(m + w)
    a = rng.standard_normal((m, w))
    t, ld = to_dev(a)
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    T = torch.zeros((w, 128), dtype=torch.float64, device="cuda")
    assert lib().qrb_op_panel(P(t), ld, m, w, P(tau), P(T), 128, None) == 0
    got = to_host(t, m)
    (qr_raw, tau_ref), _ = sla.qr(a, mode="raw")
    # same dlarfg sign convention: R, V and tau agree elementwise
    assert rel_err(np.triu(got[:w]), np.triu(qr_raw[:w])) <= 1e-12
    assert rel_err(np.tril(got, -1), np.tril(qr_raw, -1)) <= 1e-10
    np.testing.assert_allclose(tau.cpu().numpy(), tau_ref, rtol=1e-12, atol=1e-14)
    # T = the reference's forward T recurrence (kernels.py:134-147)
    v = unit_lower(got)
    taus = tau.cpu().numpy()
    t_ref = orc._t_factor(lambda k: v[:, :k].T @ v[:, k], taus)
    assert rel_err(T.cpu().numpy().T[:w, :w], t_ref) <= 1e-12


@pytest.mark.parametrize("m,w,nc", [(1000, 128, 77), (4616, 128, 5), (300, 32, 300)])
def test_apply_qt_matches_oracle(m, w, nc):
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, w))
    t, ld = to_dev(a)
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    T = torch.zeros((w, 128), dtype=torch.float64, device="cuda")
    lib().qrb_op_panel(P(t), ld, m, w, P(tau), P(T), 128, None)
    c = rng.standard_normal((m, nc))
    ct, ldc = to_dev(c)
    assert lib().qrb_op_apply_qt(P(t), ld, m, w, P(T), 128, P(ct), ldc, nc, None) == 0
    got = to_host(ct, m)
    v = unit_lower(to_host(t, m))
    tf = T.cpu().numpy().T[:w, :w]
    ref = c - v @ (tf.T @ (v.T @ c))
    assert rel_err(got, ref) <= 1e-12
    # Q^T preserves column norms
    np.testing.assert_allclose(np.linalg.norm(got, axis=0), np.linalg.norm(c, axis=0), rtol=1e-12)


@pytest.mark.parametrize("n,nb,nrhs", [(300, 128, 5), (1000, 64, 33), (128, 128, 1), (77, 16, 8)])
def test_trsm_upper(n, nb, nrhs):
    rng = np.random.default_rng(n)
    r = np.triu(rng.standard_normal((n, n))) + n * np.eye(n)
    b = rng.standard_normal((n, nrhs))
    rt, ldr = to_dev(r)
    bt, ldb = to_dev(b)
    assert lib().qrb_op_trsm_upper(P(rt), ldr, n, nb, P(bt), ldb, nrhs, None) == 0
    assert rel_err(to_host(bt, n), sla.solve_triangular(r, b)) <= 1e-12


def test_nn_dynamic_tile_schedule_is_bitwise_identical():
    """The dynamic tile tickets (multi-GPU setting) change only which CTA
    computes a tile: every C element still receives exactly one reduce-add per
    launch, so the factors are bitwise identical to the static schedule."""
    from paper_1907_01891_b200 import _native
    from paper_1907_01891_b200.device import QrDevice

    rng = np.random.default_rng(77)
    m, n = 5000, 2300
    a = rng.standard_normal((m, n))
    out = {}
    old = _native.get_tuning("nn_dynamic")
    try:
        for dyn in (0, 1):
            _native.set_tuning("nn_dynamic", dyn)
            with QrDevice(m, n) as q:
                q.set_matrix(a)
                q.factorize()
                out[dyn] = q.get_matrix()
    finally:
        _native.set_tuning("nn_dynamic", old)
    np.testing.assert_array_equal(out[0], out[1])


def test_panel_pairs_match_single_panel_steps():
    """Trailing updates with the merged 2nb-wide block reflector (outer_panels=2,
    larft merge of two panels) give the same factors as nb-wide steps."""
    from paper_1907_01891_b200 import _native
    from paper_1907_01891_b200.device import QrDevice

    rng = np.random.default_rng(12)
    m, n = 3000, 1100
    a = rng.standard_normal((m, n))
    b = rng.standard_normal((m, 4))
    res = {}
    old = _native.get_tuning("outer_panels")
    try:
        for outer in (1, 2):
            _native.set_tuning("outer_panels", outer)
            with QrDevice(m, n) as q:
                q.set_matrix(a)
                q.factorize()
                x, r, _ = q.solve(b)
                res[outer] = (q.get_matrix(), x, r)
    finally:
        _native.set_tuning("outer_panels", old)
    f1, f2 = res[1][0], res[2][0]
    assert rel_err(np.triu(f2[:n]), np.triu(f1[:n])) <= 1e-12
    assert rel_err(np.tril(f2, -1), np.tril(f1, -1)) <= 1e-11
    assert rel_err(res[2][1], res[1][1]) <= 1e-10
    np.testing.assert_allclose(res[2][2], res[1][2], rtol=1e-10)


@pytest.mark.parametrize("m,w,nb,side", [(3000, 256, 128, 0), (3000, 200, 128, 1),
                                         (5000, 100, 128, 0), (1500, 128, 64, 1)])
def test_panel_block_is_a_block_householder_qr(m, w, nb, side):
    """qrb_op_panel_block (the multi-GPU step): V (unit lower, in place), the
    merged T2 and R satisfy (I - V T2 V^T)^T A = [R; 0], with the per-panel T
    blocks on T2's diagonal; R matches LAPACK up to row signs."""
    rng = np.random.default_rng(m + w)
    a = rng.standard_normal((m, w))
    d, ld = to_dev(a)
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    tb = torch.zeros(2 * nb * nb, dtype=torch.float64, device="cuda")
    t2 = torch.zeros((w, w + (w & 1)), dtype=torch.float64, device="cuda")
    ldt2 = w + (w & 1)
    assert lib().qrb_op_panel_block(P(d), ld, m, w, nb, P(tau), P(tb), P(t2), ldt2, None,
                                    side) == 0
    f = to_host(d, m)
    T2 = t2.cpu().numpy().T[:w, :w]              # column-major (w x w)
    v = unit_lower(f)
    q = np.eye(m) - v @ T2 @ v.T
    qa = q.T @ a
    r = np.triu(f[:w])
    assert np.abs(qa[:w] - r).max() <= 1e-12 * np.abs(a).max() * np.sqrt(m)
    assert np.abs(qa[w:]).max() <= 1e-12 * np.abs(a).max() * np.sqrt(m)
    r_ref = sla.qr(a, mode="r")[0][:w]
    s = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
    assert rel_err(r * s[:, None], r_ref) <= 1e-10
    ta = tb[:nb * nb].view(nb, nb).cpu().numpy().T
    pa = min(w, nb)
    assert np.abs(T2[:pa, :pa] - ta[:pa, :pa]).max() <= 1e-14 * max(1.0, np.abs(ta).max())


@pytest.mark.parametrize("m,w,nc,split", [(3000, 256, 700, (0, 256, 300)), (2000, 128, 130, (130,)),
                                          (4000, 512, 900, (512, 100, 288))])
def test_apply_qt_two_phase_equals_apply_qt(m, w, nc, split):
    """qrb_op_apply_qt_begin + qrb_op_apply_qt_cols over any column split equals
    qrb_op_apply_qt bit for bit (the look-ahead's and the multi-GPU owner's
    update)."""
    rng = np.random.default_rng(w + nc)
    vfull = rng.standard_normal((m, w))
    t = np.triu(rng.standard_normal((w, w))) * 0.01
    c = rng.standard_normal((m, nc))
    vd, ldv = to_dev(vfull)
    td, ldt = to_dev(t)
    c1, ldc = to_dev(c)
    c2, _ = to_dev(c)
    L = lib()
    assert L.qrb_op_apply_qt(P(vd), ldv, m, w, P(td), ldt, P(c1), ldc, nc, None) == 0
    assert L.qrb_op_apply_qt_begin(P(vd), ldv, m, w, P(td), ldt, P(c2), ldc, nc, None) == 0
    c0 = 0
    for cols in split + (nc - sum(split),):
        assert L.qrb_op_apply_qt_cols(P(vd), ldv, m, w, P(c2), ldc, c0, cols, None) == 0
        c0 += cols
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    # columns beyond the last _begin are refused
    assert L.qrb_op_apply_qt_cols(P(vd), ldv, m, w, P(c2), ldc, nc, 4096, None) != 0
