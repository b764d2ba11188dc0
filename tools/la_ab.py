"""A/B of the single-GPU look-ahead (panel pair on a side stream under the
trailing update) on the BASELINE config matrices.  usage:
  python tools/la_ab.py CFG [key=value ...]   (tuning keys, e.g. la_sms=16 la_lat_us=450)
Prints factorization TFLOP/s with lookahead off and on (best of 2 after a warm-up)
and the max relative difference of R between the two."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native, ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    _native.set_tuning(k, int(v))
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
a = cs.densify_device(g, lda)
fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
q = QrDevice(m, n)
res = {}
for la in (0, 1, 0, 1):
    _native.set_tuning("lookahead", la)
    best = 0.0
    for it in range(3):
        q.set_matrix_device(a)
        s0 = _native.get_tuning("la_steps")
        rep = q.factorize()
        steps = _native.get_tuning("la_steps") - s0
        if it:
            best = max(best, fl / rep["total_ms"] / 1e9)
    r = torch.from_numpy(q.get_matrix(0, n)[:n]).triu()
    res.setdefault(la, []).append(best)
    if la == 0:
        r0 = r
    else:
        d = float((r.abs() - r0.abs()).abs().max() / r0.abs().max())
        print(f"lookahead R vs serial R (abs, max rel): {d:.2e}", flush=True)
    print(f"config {cfg} lookahead={la}: {best:.3f} TFLOP/s  ({steps} look-ahead steps)", flush=True)
print({k: max(v) for k, v in res.items()})
