"""Launch each trailing-update GEMM once at config-3 size (for ncu captures)."""
import sys, ctypes
import torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native
lib = _native.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())
M, N, K = 69120, 16384, 128
V = torch.randn(K, M, dtype=torch.float64, device="cuda")
W = torch.randn(N, 128, dtype=torch.float64, device="cuda")
C = torch.randn(N, M, dtype=torch.float64, device="cuda")
Wo = torch.zeros(N, 128, dtype=torch.float64, device="cuda")
assert lib.qrb_op_gemm_nn_sub(P(V), M, P(W), 128, P(C), M, M, N, K, None) == 0
assert lib.qrb_op_gemm_tn(P(V), M, P(C), M, P(Wo), 128, 128, N, M, 1, 1, 0, None) == 0
torch.cuda.synchronize()
print("ok")
