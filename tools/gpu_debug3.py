import sys, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native
lib = _native.load()
rng = np.random.default_rng(0)
def mk(a, ld):
    t = torch.zeros(a.shape[1], ld, dtype=torch.float64, device="cuda"); t[:, :a.shape[0]] = torch.from_numpy(a.T.copy()); return t
bad = []
for K in [16, 100, 1000, 4000, 4600, 4608, 4616, 4624, 4744, 5000, 6000, 9000]:
    for N in [5, 64, 200]:
        for M in [128, 40]:
            for splits in [1, 3]:
                A = rng.standard_normal((K, M)); B = rng.standard_normal((K, N))
                ld = (K + 31)//32*32
                At, Bt = mk(A, ld), mk(B, ld)
                Ct = torch.zeros(N, 130, dtype=torch.float64, device="cuda")
                st = lib.qrb_op_gemm_tn(ctypes.c_void_p(At.data_ptr()), ld, ctypes.c_void_p(Bt.data_ptr()), ld, ctypes.c_void_p(Ct.data_ptr()), 130, M, N, K, splits, 0, 0, None)
                torch.cuda.synchronize()
                G = Ct[:, :M].cpu().numpy().T
                err = np.abs(G - A.T @ B).max()
                if err > 1e-9 or st != 0:
                    bad.append((K, N, M, splits, err, st))
print("bad:", bad[:40])
print("count", len(bad))
