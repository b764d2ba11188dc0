"""Factors directories WRITTEN BY THE REFERENCE (oocqr.factorize), kept byte for
byte so the GPU interop test consumes real reference output, not the oracle's.

Run in the build container (where /root/reference exists):

    OOCQR_DISABLE_NUMBA=1 python tests/golden/make_golden_factors.py

For the fixture-size CT instance (config 0, 576 x 256 Siddon system, seeded
noisy sinograms) and two tilings, it runs the reference's public
factorize()/solve() and stores into ref_factors_ct0.npz: every file of the
factors directory (meta.txt, factored/, s/ incl. manifests) as raw bytes under
its relative path, the right-hand sides, and the reference's own solution X.
tests/test_gpu_interop.py re-materialises the directory and solves on the GPU.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF_SRC))
os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_cache_"))

from oocqr.task_engine import EngineConfig, factorize, solve  # noqa: E402
from oocqr.tile_store import TiledMatrix, gather_matrix, scatter_matrix  # noqa: E402

from paper_1907_01891_b200 import ct_system as cs  # noqa: E402

TILINGS = [(128, 32), (256, 64)]   # (tile_size, inner_block): 5x2 and 3x1 tile grids


def main():
    g = cs.config_geometry(0)
    a = cs.dense_matrix(g)
    x_true = cs.phantom_stack(0, 4)
    bmat = cs.noisy_sinograms(a @ x_true, 0)
    out = {"a": a, "b": bmat}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        for b, w in TILINGS:
            cfg = EngineConfig(tile_size=b, inner_block=w, cache_budget_bytes=1 << 34)
            am = TiledMatrix.create(*a.shape, b, tmp / f"a{b}")
            scatter_matrix(am, a)
            fdir = tmp / f"f{b}"
            factors, _ = factorize(am, cfg, fdir, geometry_hash=cs.geometry_hash(g))
            bm = TiledMatrix.create(*bmat.shape, b, tmp / f"b{b}")
            scatter_matrix(bm, bmat)
            xm, _ = solve(factors, bm, cfg, tmp / f"out{b}")
            out[f"t{b}_x"] = gather_matrix(xm)
            out[f"t{b}_tiling"] = np.array([b, w])
            files = sorted(p for p in fdir.rglob("*") if p.is_file())
            out[f"t{b}_paths"] = np.array([str(p.relative_to(fdir)) for p in files])
            for i, p in enumerate(files):
                out[f"t{b}_file{i}"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
    np.savez_compressed(HERE / "ref_factors_ct0.npz", **out)
    print("wrote", HERE / "ref_factors_ct0.npz")


if __name__ == "__main__":
    main()
