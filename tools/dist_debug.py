import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_1907_01891_b200 import dist as qd, ct_system as cs
from paper_1907_01891_b200.device import QrDevice
import bench
cfg = int(sys.argv[1])
g = cs.config_geometry(cfg)
coo = cs.siddon_coo(g)
m, n, nb = g.n_rays, g.n_pixels, 128
lda = (m + 31)//32*32
a_full = bench.densify_device(g, coo, lda)
a_pristine = qd.scatter_block_cyclic(a_full, n, nb, 0, 1)
print("pristine == full:", bool(torch.equal(a_pristine, a_full)), "A00", float(a_full[0, 0]), "col0 norm", float(a_full[0].norm()))
a_local = a_pristine.clone()
f = qd.factorize_distributed(a_local, m, n, nb, lda, 0, 1, qd.CudaOps())
d = torch.diagonal(f.a_local[:, :n]).cpu().numpy()
print("dist diag: min abs", np.abs(d).min(), "first", d[:4], "zeros", int((d == 0).sum()))
with QrDevice(m, n, nb) as q2:
    q2.set_matrix_device(a_pristine); q2.factorize()
    d2 = q2.rdiag()
    print("single diag first", d2[:4], "max rel diff", np.abs(np.abs(d) - np.abs(d2)).max() / np.abs(d2).max())
q = QrDevice(m, n, nb)
qd.gather_factored(f, place=lambda k, panel: q.set_matrix_device(panel, col0=k * nb))
print("placed diag first", q.rdiag()[:4])
dist.destroy_process_group()
