"""Host-staged QR at config 3 with an artificial HBM budget (development tool)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import ct_system as cs
from paper_1907_01891_b200.ooc import HostStagedQR
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
budget_gb = float(sys.argv[2]) if len(sys.argv) > 2 else 12.0
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
a_dev = cs.densify_device(g, lda)
a_host = torch.empty((n, lda), dtype=torch.float64, pin_memory=True)
a_host.copy_(a_dev)
x_true = cs.phantom_stack_device(cfg, 64)
b = (x_true @ a_dev[:, :m])
b_dev = torch.zeros((64, lda), dtype=torch.float64, device="cuda"); b_dev[:, :m] = b
del a_dev, x_true; torch.cuda.empty_cache()
q = HostStagedQR(a_host, m, n, budget_bytes=int(budget_gb * 2**30))
st = q.factorize()
t0 = time.perf_counter(); x, r = q.solve(b_dev); ts = time.perf_counter() - t0
st.update({"cfg": cfg, "budget_gb": budget_gb, "solve64_s": ts, "resid_max": float(r.max()),
           "x_max": float(x.abs().max()), "h2d_GB": st["h2d_bytes"] / 1e9})
print(json.dumps(st))
