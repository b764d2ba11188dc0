"""Per-kernel timing of the QR building blocks (development tool)."""
import sys, ctypes, os
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native
from paper_1907_01891_b200.device import QrDevice
lib = _native.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())
ev = lambda: torch.cuda.Event(enable_timing=True)

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = ev(), ev(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best

PANEL_ONLY = "--panel-only" in sys.argv
if PANEL_ONLY:
    m = int(sys.argv[-1]); w = 128
    A = torch.randn(w, m, dtype=torch.float64, device="cuda")
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    T = torch.zeros(w, w, dtype=torch.float64, device="cuda")
    A0 = A.clone()
    def f():
        A.copy_(A0)
        lib.qrb_op_panel(P(A), m, m, w, P(tau), P(T), w, None)
    print(f"panel {m}x{w}: {timeit(f):.3f} ms", flush=True)
    sys.exit(0)

for (M, N) in [(17280, 16256), (69120, 16384), (69120, 65408)]:
    K = 128
    ld = M
    V = torch.randn(K, ld, dtype=torch.float64, device="cuda")
    W = torch.randn(N, 128, dtype=torch.float64, device="cuda")
    C = torch.randn(N, ld, dtype=torch.float64, device="cuda")
    t = timeit(lambda: lib.qrb_op_gemm_nn_sub(P(V), ld, P(W), 128, P(C), ld, M, N, K, None))
    print(f"NN C-=VW {M}x{N}x{K}: {t:.2f} ms {2*M*N*K/t/1e9:.2f} TFLOP/s", flush=True)
    for splits in [1, 2]:
        Wo = torch.zeros(N, 128, dtype=torch.float64, device="cuda")
        t = timeit(lambda: lib.qrb_op_gemm_tn(P(V), ld, P(C), ld, P(Wo), 128, 128, N, M, splits, 1, 0, None))
        print(f"TN W=V^TC {128}x{N}x{M} splits={splits}: {t:.2f} ms {2*M*N*K/t/1e9:.2f} TFLOP/s", flush=True)
    del V, W, C

for m in [2160, 17280, 69120]:
    w = 128
    A = torch.randn(w, m, dtype=torch.float64, device="cuda")
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    T = torch.zeros(w, w, dtype=torch.float64, device="cuda")
    A0 = A.clone()
    def f():
        A.copy_(A0)
        lib.qrb_op_panel(P(A), m, m, w, P(tau), P(T), w, None)
    t = timeit(f)
    print(f"panel {m}x{w}: {t:.3f} ms", flush=True)

os.environ["QRB_TIMING"] = "1"
for (m, n) in [(17280, 16384)]:
    rng = np.random.default_rng(1)
    A = rng.standard_normal((m, n))
    with QrDevice(m, n) as q:
        q.set_matrix(A); rep = q.factorize()
        q.set_matrix(A); rep = q.factorize()
        f = 2*m*n*n - 2*n**3/3
        print(f"QR {m}x{n}: total {rep['total_ms']:.1f} ms panel {rep['panel_ms']:.1f} update {rep['update_ms']:.1f}  {f/rep['total_ms']/1e9:.2f} TFLOP/s launches {rep['kernel_launches']}", flush=True)
