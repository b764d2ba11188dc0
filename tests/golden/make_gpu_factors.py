"""GPU factors of the fixture-size CT instance, for the CPU test that feeds them
to the REFERENCE's own solve (tests/test_interop_cpu.py).

Run on a B200 (gpurun), from the repo root:

    python tests/golden/make_gpu_factors.py

Factors the config-0 Siddon system (576 x 256) with libqrb200 (panel width 128)
and stores the factored matrix (R + unit-lower reflectors), the per-panel T
blocks, tau, the seeded noisy sinograms and the GPU's own solution X in
gpu_factors_ct0.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402


def main():
    g = cs.config_geometry(0)
    a = cs.dense_matrix(g)
    b = cs.noisy_sinograms(a @ cs.phantom_stack(0, 4), 0)
    with QrDevice(*a.shape) as q:
        q.set_matrix(a)
        q.factorize()
        factored = q.get_matrix()
        tau, t = q.factors()
        x, resid, _ = q.solve(b)
    np.savez_compressed(HERE / "gpu_factors_ct0.npz", factored=factored, t=t, tau=tau, b=b, x=x,
                        resid=resid, nb=np.array([q.nb]))
    print("wrote", HERE / "gpu_factors_ct0.npz")


if __name__ == "__main__":
    main()
