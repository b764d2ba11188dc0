import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import ct_system as cs
from paper_1907_01891_b200.device import QrDevice
import bench
for cfg in [1, 2, 3]:
    g = cs.config_geometry(cfg)
    coo = cs.siddon_coo(g)
    m, n = g.n_rays, g.n_pixels
    lda = (m + 31)//32*32
    a = bench.densify_device(g, coo, lda)
    colnorm = torch.linalg.norm(a[:, :m], dim=1).cpu().numpy()
    with QrDevice(m, n) as q:
        q.set_matrix_device(a)
        q.factorize()
        d = np.abs(q.rdiag())
    order = np.sort(d)
    print(f"cfg{cfg}: |R_jj| max {d.max():.3e} min {d.min():.3e} ratio {d.min()/d.max():.3e}; "
          f"#<1e-6*max {np.sum(d < 1e-6*d.max())}, #<1e-10*max {np.sum(d < 1e-10*d.max())}; smallest 5 {order[:5]}; "
          f"col norms min {colnorm.min():.3e} zero cols {(colnorm==0).sum()}", flush=True)
    del a
    torch.cuda.empty_cache()
