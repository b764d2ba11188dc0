"""Golden fixture for BASELINE configuration 2 (17280 x 16384, Siddon fan-beam
A) produced by the REFERENCE package's own factorize()/solve() (run once in the
build container, ~10 min on 8 cores; the GPU test compares against it):

    OOCQR_DISABLE_NUMBA=1 python tests/golden/make_golden_cfg2.py

Stores the input sha256, X for 4 seeded noisy slices, the residual norms, |diag R|
and the first 4 rows of R (row-sign normalised) -- R itself (2 GB) is too large
to commit.  Tile size 2048, inner block 128 (the reference's
best tiling for this config).
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(HERE))
import make_golden as mg  # noqa: E402  (imports the reference from /root/reference)

from paper_1907_01891_b200 import ct_system as cs  # noqa: E402

SLICES = 4


def main():
    g = cs.config_geometry(2)
    a = cs.dense_matrix(g, order="C")
    x_true = cs.phantom_stack(2, SLICES)
    bm = cs.noisy_sinograms(a @ x_true, 2)
    t0 = time.time()
    with tempfile.TemporaryDirectory(dir=os.environ.get("GOLDEN_TMP")) as tmp:
        r, x = mg.ref_factor_solve(a, bm, 2048, 128, Path(tmp) / "ct2")
    secs = time.time() - t0
    resid = np.linalg.norm(a @ x - bm, axis=0)
    rs = mg.sign_normalise(r)
    np.savez_compressed(
        HERE / "ref_ct2.npz", a_sha256=np.array(mg.sha(a)), b_sha256=np.array(mg.sha(bm)),
        geometry_hash=np.array(cs.geometry_hash(g)), tile=np.array([2048, 128]), x=x,
        resid=resid, rdiag_abs=np.abs(np.diag(r)), r_rows4=rs[:4], b=bm,
        seconds=np.array([secs]))
    print(f"config 2 reference factorize+solve: {secs:.0f} s; |x| {np.abs(x).max():.3e}")


if __name__ == "__main__":
    main()
