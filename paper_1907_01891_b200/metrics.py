"""Image-quality and accuracy measures after the solve.

The reference's SPEC defines a ``metrics`` module (MSE, PSNR,
SSIM, relative residual) that its package never shipped.  These are the
paper's reported quantities (Tables IV/V), evaluated here
on the GPU over whole reconstructed stacks (one column per slice, images of
W x W pixels in the system-matrix column order):

* ``mse``  = mean squared error per slice                     (Eq. 5)
* ``psnr`` = 10 log10(MAX(ref)^2 / MSE), +inf when MSE = 0    (Eq. 6; MAX of
  the *reference* image)
* ``ssim`` = mean over all 8 x 8 uniform sliding windows (stride 1) of
  (2 mu_x mu_y + c1)(2 s_xy + c2) / ((mu_x^2 + mu_y^2 + c1)(s_x^2 + s_y^2 + c2)),
  c1 = (0.01 L)^2, c2 = (0.03 L)^2, L = MAX(ref)              (Eq. 7)
* ``relative_residual`` = ||A X - B||_F / ||A||_F

Window statistics are population (biased) moments of each window, computed
with box sums (2-D cumulative sums) in fp64.
"""

from __future__ import annotations

import math


def _as_images(x, w: int):
    import torch
    x = torch.as_tensor(x, dtype=torch.float64)
    if x.dim() == 1:
        x = x[:, None]
    if x.shape[0] != w * w:
        raise ValueError(f"expected {w * w} pixels per slice, got {x.shape[0]}")
    return x.T.reshape(-1, w, w)          # (slices, W, W), row 0 = +y


def mse(ref, rec, w: int):
    r, x = _as_images(ref, w), _as_images(rec, w)
    if r.shape != x.shape:
        raise ValueError(f"shape mismatch {tuple(r.shape)} vs {tuple(x.shape)}")
    return ((r - x) ** 2).mean(dim=(1, 2))


def psnr(ref, rec, w: int):
    import torch
    r = _as_images(ref, w)
    peak = r.amax(dim=(1, 2))
    if bool((peak == 0).any()):
        raise ValueError("PSNR undefined for an all-zero reference image (MAX = 0)")
    e = mse(ref, rec, w)
    out = 10.0 * torch.log10(peak ** 2 / e)
    return torch.where(e == 0, torch.full_like(out, math.inf), out)


def _box_sum(img, k: int):
    """Sum over every k x k window (stride 1): (S, W-k+1, W-k+1)."""
    import torch.nn.functional as F
    c = img.cumsum(dim=1).cumsum(dim=2)
    c = F.pad(c, (1, 0, 1, 0))
    return c[:, k:, k:] - c[:, :-k, k:] - c[:, k:, :-k] + c[:, :-k, :-k]


def ssim(ref, rec, w: int, window: int = 8, k1: float = 0.01, k2: float = 0.03,
         data_range: float | None = None):
    r, x = _as_images(ref, w), _as_images(rec, w)
    if window > w:
        raise ValueError(f"window {window} larger than the image side {w}")
    if data_range is not None:
        L = r.new_full((r.shape[0], 1, 1), float(data_range))
    else:
        L = r.amax(dim=(1, 2)).clamp_min(1e-300)[:, None, None]
    c1, c2 = (k1 * L) ** 2, (k2 * L) ** 2
    n = float(window * window)
    mr, mx = _box_sum(r, window) / n, _box_sum(x, window) / n
    vr = _box_sum(r * r, window) / n - mr * mr
    vx = _box_sum(x * x, window) / n - mx * mx
    cov = _box_sum(r * x, window) / n - mr * mx
    s = ((2 * mr * mx + c1) * (2 * cov + c2)) / ((mr * mr + mx * mx + c1) * (vr + vx + c2))
    return s.mean(dim=(1, 2))


def relative_residual(a_colmajor, x, b, m: int):
    """||A X - B||_F / ||A||_F with A a (n, lda) column-major device tensor,
    X (n x S) and B (m x S)."""
    import torch
    a = a_colmajor[:, :m]                 # (n, m) = A^T
    x = torch.as_tensor(x, dtype=torch.float64, device=a.device)
    b = torch.as_tensor(b, dtype=torch.float64, device=a.device)
    r = x.T @ a - b.T                     # (S, m)
    return float(torch.linalg.norm(r) / torch.linalg.norm(a))


def quality_report(ref, rec, w: int) -> dict:
    """Per-slice MSE / PSNR / SSIM and their averages (SPEC QualityReport)."""
    e, p, s = mse(ref, rec, w), psnr(ref, rec, w), ssim(ref, rec, w)
    return {"mse": e.tolist(), "psnr": p.tolist(), "ssim": s.tolist(),
            "mse_avg": float(e.mean()), "psnr_avg": float(p.mean()), "ssim_avg": float(s.mean())}
