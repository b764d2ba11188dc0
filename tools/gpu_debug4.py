import sys, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native
lib = _native.load()
rng = np.random.default_rng(0)
def mk(a, ld):
    t = torch.zeros(a.shape[1], ld, dtype=torch.float64, device="cuda"); t[:, :a.shape[0]] = torch.from_numpy(a.T.copy()); return t
P = lambda t: ctypes.c_void_p(t.data_ptr())
res = []
for K in [4488, 4616, 4744, 4872, 5000, 2000]:
    for N in [5, 64]:
        w = 128
        V = rng.standard_normal((K, w)) * 0.1
        Vu = np.tril(V, -1); Vu[np.arange(w), np.arange(w)] = 1.0
        T = np.triu(rng.standard_normal((w, w)))
        C = rng.standard_normal((K, N))
        ld = (K + 31)//32*32
        Vt, Ct, Tt = mk(V, ld), mk(C, ld), mk(T, 128)
        # step 1: W = Vu^T C via gemm_tn masked
        Wt = torch.zeros(N, 128, dtype=torch.float64, device="cuda")
        st1 = lib.qrb_op_gemm_tn(P(Vt), ld, P(Ct), ld, P(Wt), 128, w, N, K, 1, 1, 0, None)
        torch.cuda.synchronize()
        W = Wt.cpu().numpy().T[:w]
        e1 = np.abs(W - Vu.T @ C).max()
        # full apply
        st = lib.qrb_op_apply_qt(P(Vt), ld, K, w, P(Tt), 128, P(Ct), ld, N, None)
        torch.cuda.synchronize()
        G = Ct[:, :K].cpu().numpy().T
        ref = C - Vu @ (T.T @ (Vu.T @ C))
        e2 = np.abs(G - ref).max() / np.abs(ref).max()
        res.append((K, N, st1, e1, st, e2))
for r in res: print(r)
