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
