"""GPU solve against reference-format (tiled TD) factors."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import tiled_qr as orc
import paper_1907_01891_b200 as pkg

pytestmark = pytest.mark.gpu


def write_reference_factors(f, directory):
    """Persist oracle (= reference algorithm) factors in the reference layout
    (task_engine.py:531-594: factored/, s/, meta.txt)."""
    from paper_1907_01891_b200.interop import ReferenceFactors
    b = f.tile_size
    p = -(-f.rows // b)
    q = -(-f.cols // b)
    fac = pkg.TiledMatrix.create(f.rows, f.cols, b, directory / "factored")
    s = pkg.TiledMatrix.create(p * b, q * b, b, directory / "s")
    for (i, k), t in f.a_tiles.items():
        fac.store_tile(pkg.TileId(i, k), t)
    for (i, k), t in f.s_tiles.items():
        s.store_tile(pkg.TileId(i, k), t)
    rf = ReferenceFactors(fac, s, f.rows, f.cols, b, f.inner_block)
    rf.save(directory)
    return ReferenceFactors.load(directory)


@pytest.mark.parametrize("m,n,b,w", [(300, 200, 64, 32), (250, 250, 50, 10), (40, 24, 8, 4),
                                     (1000, 700, 256, 128)])
def test_solve_with_reference_factors(tmp_path, m, n, b, w):
    from paper_1907_01891_b200.interop import solve_reference_factors
    rng = np.random.default_rng(m + n + b)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.linspace(30, 1, n)) @ v.T
    bm = rng.standard_normal((m, 5))
    f = orc.factorize_dense(a, b, w)
    rf = write_reference_factors(f, tmp_path)
    x = solve_reference_factors(rf, bm)
    assert rel_err(x, orc.solve_dense(f, bm)) <= 1e-10


def test_reference_factors_singular_order(tmp_path, golden):
    from paper_1907_01891_b200.interop import solve_reference_factors
    z = golden("ref_singular.npz")
    b = int(z["c3_19_tile"][0])
    f = orc.factorize_dense(z["c3_19_a"], b, min(64, b))
    rf = write_reference_factors(f, tmp_path)
    with pytest.raises(pkg.SingularMatrixError) as e:
        solve_reference_factors(rf, z["c3_19_b"])
    assert e.value.global_column == int(z["c3_19_col"][0])


def _materialise(z, prefix, directory):
    """Write the oocqr-written factors directory stored byte for byte in the
    fixture (tests/golden/make_golden_factors.py) back to disk."""
    for i, rel in enumerate(z[f"{prefix}_paths"]):
        p = directory / str(rel)
        p.parent.mkdir(parents=True, exist_ok=True)
        p.write_bytes(z[f"{prefix}_file{i}"].tobytes())


@pytest.mark.parametrize("tile", [128, 256])
def test_solve_with_oocqr_written_factors(tmp_path, golden, tile):
    """Factors written by the reference's own factorize() (not the oracle):
    the GPU replay of its solve task order gives the reference's own X."""
    from paper_1907_01891_b200.interop import ReferenceFactors, solve_reference_factors
    z = golden("ref_factors_ct0.npz")
    _materialise(z, f"t{tile}", tmp_path)
    rf = ReferenceFactors.load(tmp_path)
    assert (rf.tile_size, rf.inner_block) == tuple(int(v) for v in z[f"t{tile}_tiling"])
    x = solve_reference_factors(rf, z["b"])
    assert rel_err(x, z[f"t{tile}_x"]) <= 1e-10


def test_export_roundtrip_through_reference_format(tmp_path):
    """GPU factors exported in the reference's layout (one tile, inner block =
    panel width) and replayed with the reference's solve task order give the
    GPU's own solution."""
    from paper_1907_01891_b200 import ct_system as cs
    from paper_1907_01891_b200.device import QrDevice
    from paper_1907_01891_b200.interop import (ReferenceFactors, export_reference_factors,
                                               solve_reference_factors)
    g = cs.config_geometry(1)
    a = cs.dense_matrix(g)
    b = cs.noisy_sinograms(a @ cs.phantom_stack(1, 3), 1)
    with QrDevice(*a.shape) as q:
        q.set_matrix(a)
        q.factorize()
        fac = q.get_matrix()
        _, t = q.factors()
        x_gpu, _, _ = q.solve(b)
    export_reference_factors(tmp_path, fac, t, 128, cs.geometry_hash(g))
    rf = ReferenceFactors.load(tmp_path)
    assert rf.tile_size >= a.shape[0] and rf.factored.grid_rows == 1
    x = solve_reference_factors(rf, b)
    assert rel_err(x, x_gpu) <= 1e-10
