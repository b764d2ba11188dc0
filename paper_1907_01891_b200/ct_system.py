"""Synthetic CT workloads of BASELINE.json: fan-beam Siddon system matrix,
seeded random-ellipse phantoms and noisy sinograms.

The reference builds its system matrix with Joseph's interpolating projector
(ct_model.py:223-275, 515-547) on its own Table-I geometry.  The benchmark
configurations instead specify Siddon exact intersection lengths on a simpler
geometry, which no code in the reference implements; this module is that
producer.  It keeps the reference's data layout so that image vectors line up:

* row index = view * bins + detector            (ct_model.py:535)
* column index = r * W + c, row-major pixels, image row 0 at +y
                                                (ct_model.py:245, 261, 608-612)
* ray endpoints: source at radius Rs and angle theta, flat detector at
  source-to-detector distance SDD, cell centres u_d = (d - (D-1)/2 + 1/4) * du
                                                (ct_model.py:351-360)

Geometry (recorded in :func:`geometry_hash`): square image of W x W unit
pixels centred at the origin; source radius Rs = 2 W; views uniform over
[0, 360) degrees (no quarter shift); SDD = 2 Rs; flat detector of ``bins``
cells whose fan spans the image width at the isocentre (half fan angle
asin(W / (2 Rs))), shifted by a quarter cell (the standard quarter-detector
offset).  Weights are chord lengths in pixel units (<= sqrt(2)).

Why not a fan over the whole image diagonal: BASELINE configs 2-4 have
views x bins only ~5% above the pixel count.  With the fan spanning the
circumscribed circle ~10% of the rays miss the square, the system becomes
underdetermined (measured on the GPU: 7348 of 65536 R pivots below 1e-10 of
the largest at config 3) and x is not defined.  Covering the image width puts
every ray through the image, and the quarter offset breaks the conjugate-ray
redundancy of the even view counts (90 / 180 / 720 views over 360 degrees);
on scaled analogues of configs 2-3 this gives cond(A) ~ 1e3 instead of 1e17
(tests/test_ct_system.py::test_scaled_analogue_is_well_conditioned).

The tracer is vectorised numpy (the step before the hot path, run once per
configuration); densification into the column-major device matrix happens on
the GPU from the COO triplets (see ``densify_device``).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

SEED = 190701891


@dataclass(frozen=True)
class FanGeometry:
    image_pixels: int
    views: int
    bins: int

    @property
    def source_radius(self) -> float:
        return 2.0 * self.image_pixels

    @property
    def source_to_detector(self) -> float:
        return 2.0 * self.source_radius

    @property
    def half_fan(self) -> float:
        return math.asin(self.image_pixels / (2.0 * self.source_radius))

    detector_offset = 0.25  # in cells (quarter-detector offset)

    @property
    def detector_spacing(self) -> float:
        return 2.0 * self.source_to_detector * math.tan(self.half_fan) / self.bins

    @property
    def n_rays(self) -> int:
        return self.views * self.bins

    @property
    def n_pixels(self) -> int:
        return self.image_pixels * self.image_pixels

    def angles_deg(self) -> np.ndarray:
        return 360.0 * np.arange(self.views, dtype=np.float64) / self.views


# BASELINE.json configs 1..5 (config 5 reuses config 3's matrix); 0 = test fixture size
CONFIGS = {
    0: dict(image=16, views=24, bins=24, slices=4),  # fixture-sized instance (golden vectors)
    1: dict(image=32, views=45, bins=48, slices=16),
    2: dict(image=128, views=90, bins=192, slices=64),
    3: dict(image=256, views=180, bins=384, slices=256),
    4: dict(image=512, views=720, bins=375, slices=64),
    5: dict(image=256, views=180, bins=384, slices=4096),
    # config 4's geometry family at 1/8 the image width (views/W and bins/W kept:
    # 720/512 -> 90/64, 375/512 -> 47/64; m/n = 1.03 as at full size): the
    # reduced instance the reference can factor here
    6: dict(image=64, views=90, bins=47, slices=8),
    # the same family at ~1/1.41 the width (362 x 362 image, 509 views x 265 bins:
    # A = 134885 x 131044, 141 GB -- half of config 4's rows and columns): the
    # host-staged (out-of-HBM) engine's hardware run (profiles/r02_ooc_*)
    7: dict(image=362, views=509, bins=265, slices=16),
    # the family at 1/4 the width (128 x 128 image, 180 views x 94 bins:
    # A = 16920 x 16384, m/n = 1.03): the largest instance the reference package
    # factors here in minutes (tests/golden/make_golden_cfg4q.py)
    8: dict(image=128, views=180, bins=94, slices=4),
}


def config_geometry(cfg: int) -> FanGeometry:
    c = CONFIGS[cfg]
    return FanGeometry(c["image"], c["views"], c["bins"])


def geometry_hash(g: FanGeometry) -> str:
    """Stable digest of the geometry convention (cf. ct_model.py:175-190)."""
    parts = [
        "siddon-fan-v2",
        "cover=image-width",
        f"det_offset={g.detector_offset!r}",
        f"W={g.image_pixels}",
        f"views={g.views}",
        f"bins={g.bins}",
        f"Rs={g.source_radius!r}",
        f"SDD={g.source_to_detector!r}",
        f"du={g.detector_spacing!r}",
        "angles=uniform[0,360)",
        "cols=r*W+c,row0=+y",
        "rows=view*bins+det",
    ]
    return hashlib.sha256(";".join(parts).encode()).hexdigest()[:16]


def ray_endpoints(g: FanGeometry, views: np.ndarray | None = None):
    """(sx, sy, px, py) arrays of shape (len(views), bins)."""
    if views is None:
        views = np.arange(g.views)
    theta = np.radians(360.0 * np.asarray(views, dtype=np.float64) / g.views)[:, None]
    u = ((np.arange(g.bins, dtype=np.float64) - (g.bins - 1) / 2.0 + g.detector_offset)[None, :]
         * g.detector_spacing)
    ct, st = np.cos(theta), np.sin(theta)
    sx = g.source_radius * ct + 0.0 * u
    sy = g.source_radius * st + 0.0 * u
    px = sx - g.source_to_detector * ct - u * st
    py = sy - g.source_to_detector * st + u * ct
    return sx, sy, px, py


def _siddon_block(g: FanGeometry, views: np.ndarray):
    """Siddon intersections for a block of views -> (ray, pixel, length) triplets."""
    W = g.image_pixels
    half = W / 2.0
    sx, sy, px, py = (a.ravel() for a in ray_endpoints(g, views))
    nr = sx.size
    dx, dy = px - sx, py - sy
    length = np.sqrt(dx * dx + dy * dy)
    planes = np.arange(W + 1, dtype=np.float64) - half
    with np.errstate(divide="ignore", invalid="ignore"):
        ax = (planes[None, :] - sx[:, None]) / dx[:, None]
        ay = (planes[None, :] - sy[:, None]) / dy[:, None]
    # entry / exit of the image square along the ray
    big = np.inf
    ax0 = np.where(np.abs(dx) > 0, np.minimum(ax[:, 0], ax[:, -1]), -big)
    ax1 = np.where(np.abs(dx) > 0, np.maximum(ax[:, 0], ax[:, -1]), big)
    ay0 = np.where(np.abs(dy) > 0, np.minimum(ay[:, 0], ay[:, -1]), -big)
    ay1 = np.where(np.abs(dy) > 0, np.maximum(ay[:, 0], ay[:, -1]), big)
    # a ray parallel to an axis must lie inside that slab to hit the image
    inside_x = (np.abs(dx) > 0) | ((sx > -half) & (sx < half))
    inside_y = (np.abs(dy) > 0) | ((sy > -half) & (sy < half))
    amin = np.maximum(np.maximum(ax0, ay0), 0.0)
    amax = np.minimum(np.minimum(ax1, ay1), 1.0)
    hit = inside_x & inside_y & (amax > amin)
    ax = np.where(np.isfinite(ax), ax, np.nan)
    ay = np.where(np.isfinite(ay), ay, np.nan)
    alphas = np.concatenate([amin[:, None], amax[:, None], ax, ay], axis=1)
    lo, hi = amin[:, None], amax[:, None]
    alphas = np.where((alphas >= lo) & (alphas <= hi), alphas, np.nan)
    alphas.sort(axis=1)  # NaNs sort to the end
    seg = np.diff(alphas, axis=1)
    mid = alphas[:, :-1] + 0.5 * seg
    ok = np.isfinite(seg) & (seg > 0) & hit[:, None]
    xm = sx[:, None] + mid * dx[:, None]
    ym = sy[:, None] + mid * dy[:, None]
    c = np.floor(np.where(ok, xm, 0.0) + half).astype(np.int64)
    r = np.floor(half - np.where(ok, ym, 0.0)).astype(np.int64)
    ok &= (c >= 0) & (c < W) & (r >= 0) & (r < W)
    ray_local = np.broadcast_to(np.arange(nr)[:, None], ok.shape)
    vals = seg * length[:, None]
    return ray_local[ok], (r * W + c)[ok], vals[ok]


def siddon_coo(g: FanGeometry, views_per_block: int = 16):
    """All system-matrix nonzeros as (row, col, value) int64/int64/float64 arrays,
    sorted by row (view-major) and, within a row, by distance from the source."""
    rows, cols, vals = [], [], []
    for v0 in range(0, g.views, views_per_block):
        views = np.arange(v0, min(g.views, v0 + views_per_block))
        rl, cl, vl = _siddon_block(g, views)
        rows.append(rl + v0 * g.bins)
        cols.append(cl)
        vals.append(vl)
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def densify_device(g: FanGeometry, lda: int | None = None, rank: int = 0, world: int = 1,
                   nb: int = 128, views_per_call: int = 64):
    """Dense column-major A (or this rank's block-cyclic panels) built on the GPU
    by the sm_100a Siddon kernel (qrb_siddon_densify); returns a torch tensor of
    shape (local columns, lda).  Bit-identical to :func:`dense_matrix`."""
    import torch

    m, n = g.n_rays, g.n_pixels
    lda = lda or (m + 31) // 32 * 32
    npan = -(-n // nb)
    n_local = sum(min(nb, n - k * nb) for k in range(rank, npan, world)) if world > 1 else n
    a = torch.zeros((n_local, lda), dtype=torch.float64, device="cuda")
    return densify_into(g, a, lda, rank, world, nb, views_per_call)


def densify_into(g: FanGeometry, a, lda: int, rank: int = 0, world: int = 1, nb: int = 128,
                 views_per_call: int = 64):
    """Write the Siddon weights into an already zeroed device tensor (cols, lda)."""
    import ctypes

    import torch

    from . import _native

    lib = _native.load()
    n_local = a.shape[0]
    for v0 in range(0, g.views, views_per_call):
        views = np.arange(v0, min(g.views, v0 + views_per_call))
        ends = np.stack([e.ravel() for e in ray_endpoints(g, views)])  # (4, rays)
        ends_d = torch.from_numpy(np.ascontiguousarray(ends)).cuda()
        st = lib.qrb_siddon_densify(ctypes.c_void_p(ends_d.data_ptr()), ends.shape[1],
                                    v0 * g.bins, g.image_pixels, ctypes.c_void_p(a.data_ptr()),
                                    lda, nb, world, rank, n_local, None)
        _native.check(st, "qrb_siddon_densify")
    torch.cuda.synchronize()
    return a


def dense_matrix(g: FanGeometry, order: str = "F") -> np.ndarray:
    """Dense fp64 system matrix on the host (small configurations / tests)."""
    r, c, v = siddon_coo(g)
    a = np.zeros((g.n_rays, g.n_pixels), dtype=np.float64, order=order)
    a[r, c] = v
    return a


# -- phantoms and sinograms ---------------------------------------------------


def slice_rngs(cfg: int, count: int, first: int = 0):
    """One independent generator per slice: SeedSequence(190701891, cfg) children."""
    ss = np.random.SeedSequence([SEED, int(cfg)])
    children = ss.spawn(first + count)[first:]
    return [np.random.default_rng(s) for s in children]


def random_ellipses(rng: np.random.Generator, W: int, count: int = 10) -> np.ndarray:
    """(count, 6) rows of cx, cy, a, b, theta_deg, density."""
    half = W / 2.0
    cx = rng.uniform(-half, half, count)
    cy = rng.uniform(-half, half, count)
    a = rng.uniform(0.05, 0.40, count) * W
    b = rng.uniform(0.05, 0.40, count) * W
    th = rng.uniform(0.0, 180.0, count)
    d = rng.uniform(0.0, 1.0, count)
    return np.stack([cx, cy, a, b, th, d], axis=1)


def rasterize(ellipses: np.ndarray, W: int) -> np.ndarray:
    """Additive ellipse densities sampled at pixel centres; returns the W*W
    image vector in the system-matrix column order (rasterize_phantom
    convention, ct_model.py:600-623)."""
    half = W / 2.0
    xs = np.arange(W) + 0.5 - half
    ys = half - (np.arange(W) + 0.5)
    gx, gy = np.meshgrid(xs, ys)
    img = np.zeros((W, W))
    for cx, cy, a, b, th, d in ellipses:
        t = math.radians(th)
        ddx, ddy = gx - cx, gy - cy
        u = math.cos(t) * ddx + math.sin(t) * ddy
        w = -math.sin(t) * ddx + math.cos(t) * ddy
        img[(u / a) ** 2 + (w / b) ** 2 <= 1.0] += d
    return img.ravel()


def phantom_stack(cfg: int, slices: int, first: int = 0) -> np.ndarray:
    """X_true (W*W x slices), one seeded 10-ellipse phantom per slice."""
    W = CONFIGS[cfg]["image"]
    rngs = slice_rngs(cfg, slices, first)
    return np.column_stack([rasterize(random_ellipses(r, W), W) for r in rngs])


def phantom_stack_device(cfg: int, slices: int, first: int = 0, device="cuda"):
    """Same phantoms as :func:`phantom_stack` (same per-slice RNG draws),
    rasterised on the GPU with torch: a (slices, W*W) tensor.  Used for the
    4096-slice solve-throughput workload (config 5)."""
    import torch

    W = CONFIGS[cfg]["image"]
    ell = np.stack([random_ellipses(r, W) for r in slice_rngs(cfg, slices, first)])  # (S,10,6)
    e = torch.from_numpy(ell).to(device)
    half = W / 2.0
    xs = torch.arange(W, dtype=torch.float64, device=device) + 0.5 - half
    ys = half - (torch.arange(W, dtype=torch.float64, device=device) + 0.5)
    gy, gx = torch.meshgrid(ys, xs, indexing="ij")
    gx, gy = gx.reshape(1, -1), gy.reshape(1, -1)
    img = torch.zeros((slices, W * W), dtype=torch.float64, device=device)
    for i in range(e.shape[1]):
        cx, cy, a, b, th, d = (e[:, i, k:k + 1] for k in range(6))
        t = torch.deg2rad(th)
        dx, dy = gx - cx, gy - cy
        u = torch.cos(t) * dx + torch.sin(t) * dy
        w = -torch.sin(t) * dx + torch.cos(t) * dy
        img += torch.where((u / a) ** 2 + (w / b) ** 2 <= 1.0, d, torch.zeros_like(d))
    return img


def noisy_sinograms(a_times_x: np.ndarray, cfg: int, first: int = 0) -> np.ndarray:
    """b = A x + eps, eps ~ N(0, (0.01 * max(A x))^2) per slice (seeded)."""
    ax = np.asarray(a_times_x, dtype=np.float64)
    if ax.ndim == 1:
        ax = ax[:, None]
    out = np.empty_like(ax)
    ss = np.random.SeedSequence([SEED, int(cfg), 1])
    children = ss.spawn(first + ax.shape[1])[first:]
    for j in range(ax.shape[1]):
        rng = np.random.default_rng(children[j])
        sigma = 0.01 * float(ax[:, j].max())
        out[:, j] = ax[:, j] + rng.normal(0.0, sigma, ax.shape[0])
    return out


def sparse_matvec(coo, x: np.ndarray, n_rows: int) -> np.ndarray:
    """A @ X from COO triplets without densifying (host)."""
    r, c, v = coo
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    out = np.zeros((n_rows, x.shape[1]))
    np.add.at(out, r, v[:, None] * x[c])
    return out


def workload(cfg: int, slices: int | None = None):
    """(geometry, coo, X_true, B) for a BASELINE configuration (host arrays)."""
    g = config_geometry(cfg)
    s = CONFIGS[cfg]["slices"] if slices is None else slices
    coo = siddon_coo(g)
    x = phantom_stack(cfg, s)
    b = noisy_sinograms(sparse_matvec(coo, x, g.n_rays), cfg)
    return g, coo, x, b
