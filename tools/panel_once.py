import sys, ctypes, torch
sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native
lib = _native.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())
m = int(sys.argv[1]); w = int(sys.argv[2]) if len(sys.argv) > 2 else 128
A = torch.randn(w, m, dtype=torch.float64, device="cuda")
tau = torch.zeros(w, dtype=torch.float64, device="cuda")
T = torch.zeros(w, 128, dtype=torch.float64, device="cuda")
assert lib.qrb_op_panel(P(A), m, m, w, P(tau), P(T), 128, None) == 0
torch.cuda.synchronize(); print("ok")
