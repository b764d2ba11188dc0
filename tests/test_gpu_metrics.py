"""Image-quality metrics (metrics.py) evaluated on the GPU
over reconstructed slice stacks, against per-slice naive numpy evaluations."""

import numpy as np
import pytest

from test_metrics import naive_ssim

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_metrics_on_device_stack_match_naive():
    from paper_1907_01891_b200 import ct_system as cs
    from paper_1907_01891_b200 import metrics
    from paper_1907_01891_b200.device import QrDevice

    g = cs.config_geometry(1)
    w = g.image_pixels
    a = cs.dense_matrix(g)
    x_true = cs.phantom_stack(1, 6)                      # (n, 6)
    b = cs.noisy_sinograms(a @ x_true, 1)
    with QrDevice(*a.shape) as q:
        q.set_matrix(a)
        q.factorize()
        x, _, _ = q.solve(b)
    ref_d = torch.from_numpy(x_true).cuda()
    rec_d = torch.from_numpy(x).cuda()
    mse = metrics.mse(ref_d, rec_d, w)
    psnr = metrics.psnr(ref_d, rec_d, w)
    ssim = metrics.ssim(ref_d, rec_d, w)
    assert mse.is_cuda and psnr.is_cuda and ssim.is_cuda
    for j in range(x.shape[1]):
        r = x_true[:, j].reshape(w, w)
        e = x[:, j].reshape(w, w)
        m_ref = float(((r - e) ** 2).mean())
        assert float(mse[j]) == pytest.approx(m_ref, rel=1e-12)
        assert float(psnr[j]) == pytest.approx(10 * np.log10(r.max() ** 2 / m_ref), rel=1e-12)
        assert float(ssim[j]) == pytest.approx(naive_ssim(r, e), rel=1e-9, abs=1e-12)
    # relative residual with A resident on the device (column-major (n, lda) storage)
    a_cm = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    rr = metrics.relative_residual(a_cm, rec_d, torch.from_numpy(b).cuda(), a.shape[0])
    ref_rr = np.linalg.norm(a @ x - b) / np.linalg.norm(a)
    assert rr == pytest.approx(ref_rr, rel=1e-10)
