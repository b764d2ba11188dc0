import sys, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200.device import QrDevice
from paper_1907_01891_b200 import _native
lib = _native.load()
rng = np.random.default_rng(0)
P = lambda t: ctypes.c_void_p(t.data_ptr())

for (m, n, nrhs) in [(5000, 3000, 5), (5000, 1000, 5), (3000, 2000, 5), (4000, 3000, 5), (5000, 2048, 5), (2176, 2048, 5)]:
    A = rng.standard_normal((m, n))
    B = rng.standard_normal((m, nrhs))
    with QrDevice(m, n) as q:
        q.set_matrix(A); q.factorize()
        F = q.get_matrix(); tau, Tall = q.factors()
    ld = (m + 31) // 32 * 32
    Fd = torch.zeros(n, ld, dtype=torch.float64, device="cuda"); Fd[:, :m] = torch.from_numpy(F.T.copy())
    Td = torch.from_numpy(np.ascontiguousarray(Tall.T)).cuda()  # (npanels*nb, nb) rows = columns of T
    Bd = torch.zeros(nrhs, ld, dtype=torch.float64, device="cuda"); Bd[:, :m] = torch.from_numpy(B.T.copy())
    C = B.copy()
    nb = 128
    first_bad = None
    for k in range(-(-n // nb)):
        j0 = k * nb; pw = min(nb, n - j0); mk = m - j0
        V = np.tril(F[j0:, j0:j0 + pw], -1); V[np.arange(pw), np.arange(pw)] = 1.0
        Th = Tall[:pw, k*nb:k*nb+pw]
        C[j0:] -= V @ (Th.T @ (V.T @ C[j0:]))
        vptr = Fd.data_ptr() + 8 * (j0 + j0 * ld)
        tptr = Td.data_ptr() + 8 * (k * nb * nb)
        cptr = Bd.data_ptr() + 8 * j0
        st = lib.qrb_op_apply_qt(ctypes.c_void_p(vptr), ld, mk, pw, ctypes.c_void_p(tptr), nb, ctypes.c_void_p(cptr), ld, nrhs, None)
        torch.cuda.synchronize()
        G = Bd[:, :m].cpu().numpy().T
        err = np.abs(G - C).max() / np.abs(C).max()
        if err > 1e-12 and first_bad is None:
            first_bad = (k, mk, err, st)
            rows = np.nonzero(np.abs(G - C).max(axis=1) > 1e-10 * np.abs(C).max())[0]
            print(f"   bad rows at panel {k}: count {rows.size} first {rows[:8]} last {rows[-4:]}")
            Bd[:, :m] = torch.from_numpy(C.T.copy())
    print(f"{m}x{n}: first bad panel {first_bad}", flush=True)
