"""Per-kernel-family breakdown of the multi-slice solve (development tool).
usage: python tools/solve_profile.py CFG SLICES..."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

cfg = int(sys.argv[1])
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
a = cs.densify_device(g, lda)
q = QrDevice(m, n)
q.set_matrix_device(a)
del a
torch.cuda.empty_cache()
q.factorize()
q.set_profiling(True)
for s in [int(x) for x in sys.argv[2:]]:
    b = torch.randn((s, lda), dtype=torch.float64, device="cuda")
    x = torch.zeros((s, n + (n & 1)), dtype=torch.float64, device="cuda")
    q.solve_device(b, x)
    rep = q.solve_device(b, x)
    fl = (4.0 * m * n - n * n) * s
    print(f"S={s}: {rep['total_ms']:.1f} ms  {s / rep['total_ms'] * 1e3:.0f} slices/s  "
          f"{fl / rep['total_ms'] / 1e9:.1f} TFLOP/s  launches {rep['kernel_launches']}")
    for k, v in sorted(rep["kernels"].items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {k:8s} {v['ms']:8.2f} ms  {v['flops'] / max(v['ms'], 1e-9) / 1e9:6.1f} TF  "
              f"launches {v['launches']}")
