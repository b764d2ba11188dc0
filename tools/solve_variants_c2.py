import sys, json, torch, numpy as np
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native, ct_system as cs
from paper_1907_01891_b200.device import QrDevice
g = cs.config_geometry(2); m, n = g.n_rays, g.n_pixels; lda = (m + 31)//32*32
a = cs.densify_device(g, lda)
S = 64
b = torch.randn((S, lda), dtype=torch.float64, device="cuda"); x = torch.zeros((S, n), dtype=torch.float64, device="cuda")
for name, knobs in [("singles_nomerge", {"outer_panels": 0, "t4_min_rhs": 1024}), ("singles_merge", {"outer_panels": 0, "t4_min_rhs": 0}), ("pairs", {"outer_panels": 2, "t4_min_rhs": 1024}), ("auto4", {"outer_panels": 4, "t4_min_rhs": 1024})]:
    for k, v in knobs.items(): _native.set_tuning(k, v)
    q = QrDevice(m, n); fs, ss = [], []
    for it in range(4):
        q.set_matrix_device(a); f = q.factorize()["total_ms"]; s_ = q.solve_device(b, x)["total_ms"]
        if it: fs.append(f); ss.append(s_)
    q.close()
    print(json.dumps({"v": name, "factor_ms": min(fs), "solve_ms": min(ss)}), flush=True)
