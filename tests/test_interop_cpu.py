"""GPU factors in the reference's on-disk format, solved by the REFERENCE.

tests/golden/gpu_factors_ct0.npz holds a factorization produced by libqrb200
on a B200 (tests/golden/make_gpu_factors.py).  export_reference_factors writes
it as an oocqr factors directory; the reference package's own solve()
(task_engine.py:644-685) must read it and return the GPU's solution.  Needs the
reference sources (/root/reference, build container only); skipped elsewhere.
"""

import os
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def oocqr():
    if not (REF_SRC / "oocqr").is_dir():
        pytest.skip("reference sources not present (GPU box)")
    os.environ.setdefault("OOCQR_DISABLE_NUMBA", "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_cache_"))
    sys.path.insert(0, str(REF_SRC))
    import oocqr.task_engine as te
    import oocqr.tile_store as ts
    return te, ts


def test_reference_solve_reads_exported_gpu_factors(tmp_path, golden, oocqr):
    te, ts = oocqr
    from paper_1907_01891_b200.interop import export_reference_factors
    z = golden("gpu_factors_ct0.npz")
    nb = int(z["nb"][0])
    rf = export_reference_factors(tmp_path / "f", z["factored"], z["t"], nb)
    factors = te.QrFactors.load(tmp_path / "f")            # the reference's own loader
    assert (factors.tile_size, factors.inner_block) == (rf.tile_size, nb)
    b = z["b"]
    bm = ts.TiledMatrix.create(b.shape[0], b.shape[1], factors.tile_size, tmp_path / "b")
    ts.scatter_matrix(bm, b)
    cfg = te.EngineConfig(tile_size=factors.tile_size, inner_block=nb)
    xm, _ = te.solve(factors, bm, cfg, tmp_path / "out")
    x = ts.gather_matrix(xm)
    assert rel_err(x, z["x"]) <= 1e-8
    # and the reference's own factorization of the same system (another tiling)
    zr = golden("ref_factors_ct0.npz")
    np.testing.assert_array_equal(zr["b"], b)
    assert rel_err(x, zr["t128_x"]) <= 1e-8
