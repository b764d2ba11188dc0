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
ld = 5024
Fd = torch.zeros(n, ld, dtype=torch.float64, device="cuda"); Fd[:, :m] = torch.from_numpy(F.T.copy())
Td = torch.from_numpy(np.ascontiguousarray(Tall.T)).cuda()
nb = 128
for k in [2, 3, 4]:
    j0 = k*nb; pw = 128; mk = m - j0
    V = np.tril(F[j0:, j0:j0+pw], -1); V[np.arange(pw), np.arange(pw)] = 1.0
    Th = Tall[:, k*nb:(k+1)*nb]
    C = rng.standard_normal((mk, nrhs))
    Cd = torch.zeros(nrhs, ld, dtype=torch.float64, device="cuda"); Cd[:, j0:m] = torch.from_numpy(C.T.copy())
    vptr = ctypes.c_void_p(Fd.data_ptr() + 8*(j0 + j0*ld)); cptr = ctypes.c_void_p(Cd.data_ptr() + 8*j0)
    tptr = ctypes.c_void_p(Td.data_ptr() + 8*k*nb*nb)
    W = torch.zeros(nrhs, 128, dtype=torch.float64, device="cuda")
    s1 = lib.qrb_op_gemm_tn(vptr, ld, cptr, ld, P(W), 128, pw, nrhs, mk, 1, 1, 0, None); torch.cuda.synchronize()
    Wh = W.cpu().numpy().T
    e1 = np.abs(Wh - V.T @ C).max() / np.abs(V.T @ C).max()
    W2 = torch.zeros(nrhs, 128, dtype=torch.float64, device="cuda")
    s2 = lib.qrb_op_gemm_tn(tptr, nb, P(W), 128, P(W2), 128, pw, nrhs, pw, 1, 0, 0, None); torch.cuda.synchronize()
    W2h = W2.cpu().numpy().T
    e2 = np.abs(W2h - Th.T @ Wh).max() / np.abs(Th.T @ Wh).max()
    # NN: C -= V W2 (masked V) -- emulate via gemm_nn_sub with explicit V
    Vd = torch.zeros(pw, ld, dtype=torch.float64, device="cuda"); Vd[:, :mk] = torch.from_numpy(V.T.copy())
    C2 = Cd.clone()
    s3 = lib.qrb_op_gemm_nn_sub(P(Vd), ld, P(W2), 128, ctypes.c_void_p(C2.data_ptr()+8*j0), ld, mk, nrhs, pw, None); torch.cuda.synchronize()
    e3 = np.abs(C2[:, j0:m].cpu().numpy().T - (C - V @ W2h)).max()
    # full op
    C3 = Cd.clone()
    s4 = lib.qrb_op_apply_qt(vptr, ld, mk, pw, tptr, nb, ctypes.c_void_p(C3.data_ptr()+8*j0), ld, nrhs, None); torch.cuda.synchronize()
    ref = C - V @ (Th.T @ (V.T @ C))
    e4 = np.abs(C3[:, j0:m].cpu().numpy().T - ref).max() / np.abs(ref).max()
    print(k, mk, "TN(V^T C)", s1, e1, "TN(T^T W)", s2, e2, "NN", s3, e3, "apply", s4, e4, flush=True)
    print("   tau range", tau[j0:j0+pw].min(), tau[j0:j0+pw].max(), "T absmax", np.abs(Th).max(), "T lower", np.abs(np.tril(Th,-1)).max())
