"""Look-ahead knob sweep on one configuration (development tool).

python tools/la_sweep2.py CFG key=v1,v2 [key=v1,v2 ...]
Times the (graph-replayed when eligible) factorization for every combination.
"""
import itertools
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native  # noqa: E402
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

cfg = int(sys.argv[1])
REPS = 3 if cfg < 3 else 2
knobs = [(kv.split("=")[0], [int(v) for v in kv.split("=")[1].split(",")]) for kv in sys.argv[2:]]
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
a = cs.densify_device(g, (m + 31) // 32 * 32)
fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3
_native.load()
for combo in itertools.product(*[v for _, v in knobs]):
    for (k, _), v in zip(knobs, combo):
        _native.set_tuning(k, v)
    q = QrDevice(m, n)
    best = 1e30
    for it in range(REPS + 1):
        q.set_matrix_device(a)
        torch.cuda.synchronize()
        ms = q.factorize()["total_ms"]
        if it >= 1:
            best = min(best, ms)
    q.close()
    print(json.dumps({"cfg": cfg, **{k: v for (k, _), v in zip(knobs, combo)}, "ms": round(best, 3),
                      "tflops": round(fl / best / 1e9, 3)}), flush=True)
