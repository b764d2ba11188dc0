"""Quick GPU numerics + timing check of libqrb200 (development tool)."""
import sys, time, ctypes
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native
from paper_1907_01891_b200.device import QrDevice

lib = _native.load()
rng = np.random.default_rng(0)

def dev(a):  # numpy F-order (m x k) -> torch tensor (k, m) on cuda
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, order="F").T)).cuda()

def host(t):
    return t.cpu().numpy().T.copy(order="F")

def p(t):
    return ctypes.c_void_p(t.data_ptr())

# --- gemm_nn_sub vs numpy
for (m, n, k) in [(128, 64, 16), (300, 70, 37), (1000, 513, 128), (64, 8, 3)]:
    A = rng.standard_normal((m, k)); B = rng.standard_normal((k, n)); C = rng.standard_normal((m, n))
    ld = lambda x: x + (x & 1)
    At = torch.zeros(k, ld(m), dtype=torch.float64, device="cuda"); At[:, :m] = torch.from_numpy(A.T)
    Bt = torch.zeros(n, ld(k), dtype=torch.float64, device="cuda"); Bt[:, :k] = torch.from_numpy(B.T)
    Ct = torch.zeros(n, ld(m), dtype=torch.float64, device="cuda"); Ct[:, :m] = torch.from_numpy(C.T)
    st = lib.qrb_op_gemm_nn_sub(p(At), ld(m), p(Bt), ld(k), p(Ct), ld(m), m, n, k, None)
    torch.cuda.synchronize()
    got = Ct[:, :m].cpu().numpy().T
    err = np.abs(got - (C - A @ B)).max()
    print(f"gemm_nn_sub {m}x{n}x{k}: status {st} maxerr {err:.2e}", flush=True)

# --- full QR + solve
for (m, n) in [(64, 48), (300, 200), (2160, 1024), (5000, 3000)]:
    A = rng.standard_normal((m, n))
    X0 = rng.standard_normal((n, 5))
    Bm = A @ X0
    with QrDevice(m, n) as q:
        q.set_matrix(A)
        rep = q.factorize()
        R = q.r_factor()
        Rref = np.linalg.qr(A, mode="r")
        s = np.sign(np.diag(R)) * np.sign(np.diag(Rref))
        errR = np.abs(R * s[:, None] - Rref).max() / np.abs(Rref).max()
        X, res, srep = q.solve(Bm)
        errX = np.abs(X - X0).max() / np.abs(X0).max()
        print(f"QR {m}x{n}: R relerr {errR:.2e}  X relerr {errX:.2e}  resid {res.max():.2e}  "
              f"factor {rep['total_ms']:.2f} ms launches {rep['kernel_launches']}", flush=True)

# --- timing of a config-2 sized QR
for (m, n) in [(17280, 16384)]:
    A = rng.standard_normal((m, n))
    with QrDevice(m, n) as q:
        for it in range(2):
            q.set_matrix(A)
            rep = q.factorize()
        f = 2*m*n*n - 2*n**3/3
        print(f"QR {m}x{n}: {rep['total_ms']:.1f} ms  {f/rep['total_ms']/1e9:.2f} TFLOP/s", flush=True)
        Rref_d = None
        B = rng.standard_normal((m, 64))
        X, res, srep = q.solve(B)
        print(f"solve 64: {srep['total_ms']:.2f} ms, update {srep['update_ms']:.2f}", flush=True)
        Xref = np.linalg.lstsq(A, B, rcond=None)[0]
        print(f"solve relerr vs lstsq {np.abs(X-Xref).max()/np.abs(Xref).max():.2e}", flush=True)
