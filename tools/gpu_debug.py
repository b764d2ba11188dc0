import sys, ctypes
import numpy as np
sys.path.insert(0, ".")
from paper_1907_01891_b200.device import QrDevice

rng = np.random.default_rng(0)

def build_t_host(V, tau):
    w = V.shape[1]
    T = np.zeros((w, w))
    for k in range(w):
        T[k, k] = tau[k]
        if k > 0 and tau[k] != 0:
            z = V[:, :k].T @ V[:, k]
            T[:k, k] = -tau[k] * (T[:k, :k] @ z)
    return T

for (m, n, nrhs) in [(2160, 1024, 5), (5000, 3000, 5), (5000, 3000, 64), (3000, 3000, 5), (4000, 1000, 5)]:
    A = rng.standard_normal((m, n))
    B = rng.standard_normal((m, nrhs))
    with QrDevice(m, n) as q:
        q.set_matrix(A)
        q.factorize()
        F = q.get_matrix()
        tau, Tall = q.factors()
        X, res, _ = q.solve(B)
    nb = 128
    C = B.copy()
    worst_t = 0
    for k in range(-(-n // nb)):
        j0 = k * nb; pw = min(nb, n - j0)
        V = np.tril(F[j0:, j0:j0 + pw], -1)
        V[np.arange(pw), np.arange(pw)] = 1.0
        Th = build_t_host(V, tau[j0:j0 + pw])
        Tg = Tall[:pw, k * nb:k * nb + pw]
        et = np.abs(Th - Tg).max() / max(np.abs(Th).max(), 1e-300)
        if et > worst_t:
            worst_t = et; wk = k
        C[j0:] -= V @ (Th.T @ (V.T @ C[j0:]))
    R = np.triu(F[:n])
    Xh = np.linalg.solve(R, C[:n])
    resh = np.linalg.norm(C[n:], axis=0)
    Xref = np.linalg.lstsq(A, B, rcond=None)[0]
    print(f"{m}x{n} nrhs={nrhs}: worst T relerr {worst_t:.2e} (panel {wk}); host-apply X err {np.abs(Xh-Xref).max():.2e}; "
          f"gpu X err {np.abs(X-Xref).max():.2e}; resid host {resh.max():.3e} gpu {res.max():.3e}", flush=True)
