"""NN trailing-update GEMM throughput as a function of K (development tool)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native  # noqa: E402

lib = _native.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


M, N = 69120, 32768
for K in [128, 256, 384, 512]:
    V = torch.randn(K, M, dtype=torch.float64, device="cuda")
    W = torch.randn(N, K, dtype=torch.float64, device="cuda")
    C = torch.randn(N, M, dtype=torch.float64, device="cuda")
    t = timeit(lambda: lib.qrb_op_gemm_nn_sub(P(V), M, P(W), K, P(C), M, M, N, K, None))
    tn = torch.zeros(N, K, dtype=torch.float64, device="cuda")
    t2 = timeit(lambda: lib.qrb_op_gemm_tn(P(V), M, P(C), M, P(tn), K, K, N, M, 1, 0, 0, None))
    print(f"K={K}: NN {2 * M * N * K / t / 1e9:.2f} TFLOP/s   TN {2 * M * N * K / t2 / 1e9:.2f} TFLOP/s",
          flush=True)
    del V, W, C, tn
