"""qrb_factorize_host at config 3 for several chunk widths (development tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

g = cs.config_geometry(3)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
a = cs.densify_device(g, lda)
pin = torch.empty((n, lda), dtype=torch.float64, pin_memory=True)
pin.copy_(a)
del a
torch.cuda.empty_cache()
view = pin.numpy().T[:m, :]
fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3
with QrDevice(m, n) as q:
    for chunk in [int(x) for x in sys.argv[1:]]:
        t0 = time.perf_counter()
        rep = q.factorize_host(view, chunk_cols=chunk)
        wall = time.perf_counter() - t0
        print(f"chunk {chunk}: {rep['total_ms']:.0f} ms ({fl / rep['total_ms'] / 1e9:.2f} TFLOP/s), "
              f"h2d {rep['h2d_ms']:.0f} ms, wall {wall * 1e3:.0f} ms", flush=True)
