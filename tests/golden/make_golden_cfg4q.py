"""Golden fixture for the config-4 geometry family at 1/4 width (ct_system
CONFIGS[8]: 128 x 128 image, 180 views x 94 bins -> A = 16920 x 16384, m/n =
1.03 like config 4's 270000 x 262144) from the REFERENCE package's own
factorize()/solve() (tile 2048, inner block 128):

    OOCQR_DISABLE_NUMBA=1 python tests/golden/make_golden_cfg4q.py

Config 4 itself (566 GB) cannot be factored by the reference here; this pins
its family at the largest size the reference finishes in minutes (the 1/8
width fixture ref_ct4r.npz is the small one).  Stores X for 4 noisy slices,
the residual norms, |diag R|, the first 8 rows of R (row-sign normalised) and
the input sha256.
"""

from __future__ import annotations

import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as mg  # noqa: E402  (imports the reference from /root/reference)

from paper_1907_01891_b200 import ct_system as cs  # noqa: E402

CFG = 8


def main():
    g = cs.config_geometry(CFG)
    a = cs.dense_matrix(g, order="C")
    s = cs.CONFIGS[CFG]["slices"]
    x_true = cs.phantom_stack(CFG, s)
    bm = cs.noisy_sinograms(a @ x_true, CFG)
    t0 = time.time()
    with tempfile.TemporaryDirectory() as tmp:
        r, x = mg.ref_factor_solve(a, bm, 2048, 128, Path(tmp) / "ct4q")
    secs = time.time() - t0
    resid = np.linalg.norm(a @ x - bm, axis=0)
    rs = mg.sign_normalise(r)
    np.savez_compressed(
        HERE / "ref_ct4q.npz", a_sha256=np.array(mg.sha(a)), b_sha256=np.array(mg.sha(bm)),
        geometry_hash=np.array(cs.geometry_hash(g)), tile=np.array([2048, 128]), x=x,
        resid=resid, rdiag_abs=np.abs(np.diag(r)), r_rows8=rs[:8], b=bm, x_true=x_true,
        seconds=np.array([secs]))
    print(f"quarter-width config-4 family reference factorize+solve: {secs:.1f} s")


if __name__ == "__main__":
    main()
