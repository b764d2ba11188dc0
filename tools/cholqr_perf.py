"""Panel algorithm comparison: Householder columns vs CholeskyQR2 (development tool)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

lib = _native.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def timeit(fn, reps=5):
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


for m in [2160, 4096, 8192, 17280, 34560, 69120]:
    w = 128
    A = torch.randn(w, m, dtype=torch.float64, device="cuda")
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    T = torch.zeros(w, w, dtype=torch.float64, device="cuda")
    A0 = A.clone()
    res = {}
    for algo in (1, 2):
        _native.set_tuning("panel_algo", algo)

        def f():
            A.copy_(A0)
            lib.qrb_op_panel(P(A), m, m, w, P(tau), P(T), w, None)
        res[algo] = timeit(f)
    print(f"panel {m}x{w}: householder {res[1]:.3f} ms  cholqr2 {res[2]:.3f} ms", flush=True)

for (m, n) in [(17280, 16384), (69120, 65536)]:
    if m * n * 8 > 40e9:
        continue
    A = torch.randn(n, m, dtype=torch.float64, device="cuda")
    for algo in (1, 0):
        _native.set_tuning("panel_algo", algo)
        with QrDevice(m, n) as q:
            q.set_profiling(True)
            q.set_matrix_device(A)
            q.factorize()
            q.set_matrix_device(A)
            rep = q.factorize()
            f = 2 * m * n * n - 2 * n ** 3 / 3
            print(f"QR {m}x{n} algo {algo}: total {rep['total_ms']:.1f} ms panel "
                  f"{rep['panel_ms']:.1f} update {rep['update_ms']:.1f} "
                  f"{f / rep['total_ms'] / 1e9:.2f} TFLOP/s fallbacks "
                  f"{_native.get_tuning('cholqr_fallbacks')}", flush=True)
    del A
