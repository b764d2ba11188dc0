import sys, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200.device import QrDevice
from paper_1907_01891_b200 import _native
lib = _native.load()
rng = np.random.default_rng(0)
P = lambda t: ctypes.c_void_p(t.data_ptr())
m, n, nrhs = 5000, 1000, 5
A = rng.standard_normal((m, n)); B = rng.standard_normal((m, nrhs))
with QrDevice(m, n) as q:
    q.set_matrix(A); q.factorize()
    F = q.get_matrix(); tau, Tall = q.factors()
ld = 5024; nb = 128
Fd = torch.zeros(n, ld, dtype=torch.float64, device="cuda"); Fd[:, :m] = torch.from_numpy(F.T.copy())
Td = torch.from_numpy(np.ascontiguousarray(Tall.T)).cuda()
C = B.copy()
Bd = torch.zeros(nrhs, ld, dtype=torch.float64, device="cuda"); Bd[:, :m] = torch.from_numpy(B.T.copy())
for k in range(5):
    j0 = k*nb; pw = 128; mk = m - j0
    V = np.tril(F[j0:, j0:j0+pw], -1); V[np.arange(pw), np.arange(pw)] = 1.0
    Th = Tall[:, k*nb:(k+1)*nb]
    vptr = ctypes.c_void_p(Fd.data_ptr() + 8*(j0 + j0*ld)); cptr = ctypes.c_void_p(Bd.data_ptr() + 8*j0)
    tptr = ctypes.c_void_p(Td.data_ptr() + 8*k*nb*nb)
    Cj = C[j0:].copy()
    W = torch.zeros(nrhs, 128, dtype=torch.float64, device="cuda")
    s1 = lib.qrb_op_gemm_tn(vptr, ld, cptr, ld, P(W), 128, pw, nrhs, mk, 1, 1, 0, None); torch.cuda.synchronize()
    Wh = W.cpu().numpy().T
    e1 = np.abs(Wh - V.T @ Cj).max() / np.abs(V.T @ Cj).max()
    Gin = Bd[:, j0:m].cpu().numpy().T
    e0 = np.abs(Gin - Cj).max()
    C[j0:] -= V @ (Th.T @ (V.T @ C[j0:]))
    s4 = lib.qrb_op_apply_qt(vptr, ld, mk, pw, tptr, nb, cptr, ld, nrhs, None); torch.cuda.synchronize()
    G = Bd[:, :m].cpu().numpy().T
    e4 = np.abs(G - C).max() / np.abs(C).max()
    print(k, mk, "input err", e0, "TN", e1, "apply", e4, flush=True)
    if e1 > 1e-12:
        diff = np.abs(Wh - V.T @ Cj)
        print("  W bad entries (row, col):", np.argwhere(diff > 1e-10 * np.abs(V.T @ Cj).max())[:20].tolist())
        # recompute with explicit V to isolate masking
        Vd = torch.zeros(pw, ld, dtype=torch.float64, device="cuda"); Vd[:, :mk] = torch.from_numpy(V.T.copy())
        W3 = torch.zeros(nrhs, 128, dtype=torch.float64, device="cuda")
        lib.qrb_op_gemm_tn(P(Vd), ld, cptr, ld, P(W3), 128, pw, nrhs, mk, 1, 0, 0, None); torch.cuda.synchronize()
        print("  explicit-V TN err", np.abs(W3.cpu().numpy().T - V.T @ Cj).max())
        raw = F[j0:, j0:j0+pw]
        Vraw_d = torch.zeros(pw, ld, dtype=torch.float64, device="cuda"); Vraw_d[:, :mk] = torch.from_numpy(raw.T.copy())
        W4 = torch.zeros(nrhs, 128, dtype=torch.float64, device="cuda")
        lib.qrb_op_gemm_tn(P(Vraw_d), ld, cptr, ld, P(W4), 128, pw, nrhs, mk, 1, 1, 0, None); torch.cuda.synchronize()
        print("  raw-copy masked TN err", np.abs(W4.cpu().numpy().T - V.T @ Cj).max())
        print("  F device vs host diff:", np.abs(Fd[j0:j0+pw, j0:m].cpu().numpy().T - raw).max())
