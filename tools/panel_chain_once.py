"""One panel-pair chain (qrb_op_panel_block, m x 2nb) inside a profiler range,
for an ncu launch list of the chain (run under ncu --profile-from-start off):

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --csv python tools/panel_chain_once.py 69120
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 69120
nb, w = 128, 256
lib = _native.load()
ld = m + (m & 1)
a0 = torch.randn((w, ld), dtype=torch.float64, device="cuda")
a = torch.empty_like(a0)
tau = torch.zeros(w, dtype=torch.float64, device="cuda")
t = torch.zeros((2, nb, nb), dtype=torch.float64, device="cuda")
t2 = torch.zeros((w, w), dtype=torch.float64, device="cuda")
P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
for it in range(3):
    a.copy_(a0)
    torch.cuda.synchronize()
    if it == 2:
        torch.cuda.cudart().cudaProfilerStart()
    _native.check(lib.qrb_op_panel_block(P(a), ld, m, w, nb, P(tau), P(t), P(t2), w, None, 0),
                  "qrb_op_panel_block")
    torch.cuda.synchronize()
    if it == 2:
        torch.cuda.cudart().cudaProfilerStop()
print("done")
