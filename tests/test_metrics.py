"""Image-quality metrics (SPEC.md:401-463 examples) on CPU tensors."""

import math

import numpy as np
import pytest
import torch

from paper_1907_01891_b200 import metrics


def col(img):
    return np.asarray(img, dtype=np.float64).reshape(-1, 1)


def test_mse_examples():
    assert float(metrics.mse(col(np.eye(4)), col(np.eye(4)), 4)[0]) == 0.0
    assert float(metrics.mse(col(np.zeros((3, 3))), col(np.ones((3, 3))), 3)[0]) == 1.0
    ref = [[0.0, 2.0], [0.0, 2.0]]
    assert float(metrics.mse(col(ref), col(np.ones((2, 2))), 2)[0]) == 1.0


def test_psnr_examples():
    rng = np.random.default_rng(0)
    img = rng.random((8, 8))
    assert math.isinf(float(metrics.psnr(col(img), col(img), 8)[0]))
    ref = np.zeros((4, 4))
    ref[0, 0] = 255.0
    rec = ref.copy()
    rec += 1.0  # MSE = 1
    assert float(metrics.psnr(col(ref), col(rec), 4)[0]) == pytest.approx(48.1308, abs=1e-4)
    with pytest.raises(ValueError):
        metrics.psnr(col(np.zeros((4, 4))), col(np.ones((4, 4))), 4)


def naive_ssim(r, x, k=8, L=None):
    L = r.max() if L is None else L
    c1, c2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    vals = []
    for i in range(r.shape[0] - k + 1):
        for j in range(r.shape[1] - k + 1):
            a, b = r[i:i + k, j:j + k], x[i:i + k, j:j + k]
            ma, mb = a.mean(), b.mean()
            va, vb = a.var(), b.var()
            cv = ((a - ma) * (b - mb)).mean()
            vals.append((2 * ma * mb + c1) * (2 * cv + c2) / ((ma ** 2 + mb ** 2 + c1) * (va + vb + c2)))
    return float(np.mean(vals))


def test_ssim_examples_and_naive_agreement():
    rng = np.random.default_rng(1)
    img = rng.random((16, 16))
    assert float(metrics.ssim(col(img), col(img), 16)[0]) == pytest.approx(1.0, abs=1e-12)
    # SPEC example: constant 0 reference, reference + 1, L = 1 -> c1 / (1 + c1)
    z = np.zeros((8, 8))
    c1 = 1e-4
    got = float(metrics.ssim(col(z), col(z + 1.0), 8, data_range=1.0)[0])
    assert got == pytest.approx(c1 / (1 + c1), rel=1e-9)
    rec = img + 0.05 * rng.standard_normal((16, 16))
    assert float(metrics.ssim(col(img), col(rec), 16)[0]) == pytest.approx(naive_ssim(img, rec),
                                                                           rel=1e-10)
    with pytest.raises(ValueError):
        metrics.ssim(col(np.eye(4)), col(np.eye(4)), 4)


def test_relative_residual():
    rng = np.random.default_rng(2)
    m, n = 30, 20
    a = rng.standard_normal((m, n))
    x = rng.standard_normal((n, 3))
    a_cm = torch.from_numpy(np.ascontiguousarray(a.T))     # (n, m) column-major storage
    assert metrics.relative_residual(a_cm, np.zeros((n, 3)), np.zeros((m, 3)), m) == 0.0
    assert metrics.relative_residual(a_cm, x, a @ x, m) <= 1e-14
    rep = metrics.quality_report(col(np.eye(8)), col(np.eye(8) * 0.99), 8)
    assert rep["ssim_avg"] > 0.99 and rep["mse_avg"] > 0
