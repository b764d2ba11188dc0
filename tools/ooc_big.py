"""Host-staged (out-of-HBM) QR + solve of a large CT system on one B200, with
parity checks that need no second copy of A (run on the GPU box):

    python tools/ooc_big.py CFG BUDGET_GB [SLICES]

A (column-major, lda = m rounded to 32) is densified on the GPU by the Siddon
kernel, copied into page-locked host memory (numpy + cudaHostRegister: the torch
pinned allocator rounds to powers of two) and factored by HostStagedQR with at
most BUDGET_GB of HBM for the super-panel.  Then SLICES noisy sinograms are
solved.  Checks (A is re-densified block by block on the GPU, never stored twice):
  * residual identity  ||A x - b|| (explicit) == ||(Q^T b)[n:m]|| (from the solve)
  * sampled Gram columns (A^T A)[:, J] == (R^T R)[:, J] for 16 seeded columns J
  * noiseless recovery: x from A x_true reproduces x_true
Prints one JSON line (TFLOP/s, PCIe bytes vs the super-panel model, clocks, checks).
"""
import ctypes
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.ooc import HostStagedQR  # noqa: E402

cfg = int(sys.argv[1])
budget = int(float(sys.argv[2]) * 2**30)
S = int(sys.argv[3]) if len(sys.argv) > 3 else 16
BLK = 8192                        # columns per re-densified block in the checks
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
nb = 128
out = {"cfg": cfg, "m": m, "n": n, "a_gb": 8 * lda * n / 1e9, "budget_gb": budget / 2**30}
t0 = time.perf_counter()

# -- A on the GPU, then page-locked host memory -----------------------------------------
a_dev = cs.densify_device(g, lda)
x_true = cs.phantom_stack_device(cfg, S)                       # (S, n)
ax = x_true @ a_dev[:, :m]                                      # (S, m)
b_host = cs.noisy_sinograms(ax.cpu().numpy().T, cfg)           # (m, S)
out["densify_s"] = time.perf_counter() - t0
host_np = np.empty((n, lda), dtype=np.float64)
cudart = torch.cuda.cudart()
rc = cudart.cudaHostRegister(host_np.ctypes.data, host_np.nbytes, 0)
assert int(rc) == 0, f"cudaHostRegister failed: {rc}"
a_host = torch.from_numpy(host_np)
a_host.copy_(a_dev)
del a_dev
torch.cuda.synchronize()
torch.cuda.empty_cache()
out["stage_in_s"] = time.perf_counter() - t0

# -- factorization ----------------------------------------------------------------------
q = HostStagedQR(a_host, m, n, nb=nb, budget_bytes=budget)
clk = ClockSampler()
clk.start()
st = q.factorize()
clocks = clk.stop()
out.update({"factor_s": st["seconds"], "tflops": st["tflops"], "clocks": clocks,
            "super_panels": st["super_panels"], "super_panel_cols": st["super_panel_cols"],
            "in_core_s": st["in_core_s"], "pcie_h2d_gb": st["h2d_bytes"] / 1e9,
            "pcie_d2h_gb": st["d2h_bytes"] / 1e9, "v_stream_gb": st["v_stream_bytes"] / 1e9})
# super-panel model: S in and out once, plus every earlier panel's reflectors per super-panel
sp = st["super_panel_cols"]
model_v = sum(8 * (m - k * nb) * min(nb, n - k * nb) for c0 in range(0, n, sp)
              for k in range(c0 // nb))
out["pcie_model_gb"] = {"panels_in": 8 * lda * n / 1e9, "panels_out": 8 * lda * n / 1e9,
                        "reflectors": model_v / 1e9}

# -- solve --------------------------------------------------------------------------------
b_dev = torch.zeros((S, lda), dtype=torch.float64, device="cuda")
b_dev[:, :m] = torch.from_numpy(np.ascontiguousarray(b_host.T)).cuda()
torch.cuda.synchronize()
ts = time.perf_counter()
x, resid = q.solve(b_dev)
torch.cuda.synchronize()
out["solve_s"] = time.perf_counter() - ts
out["slices_per_s"] = S / out["solve_s"]
b0 = torch.zeros_like(b_dev)
b0[:, :m] = ax
x0, _ = q.solve(b0)
out["noiseless_x_rel_err"] = float((torch.linalg.norm(x0 - x_true, dim=1)
                                    / torch.linalg.norm(x_true, dim=1)).max())


# -- checks against A re-densified block by block ------------------------------------------
def a_block(c0, w):
    """Columns [c0, c0 + w) of A on the device (cols, lda): the densifier's
    block-cyclic mode with one block per 'rank' (panel width = block width)."""
    nblk = -(-n // BLK)
    t = torch.zeros((w, lda), dtype=torch.float64, device="cuda")
    return cs.densify_into(g, t, lda, rank=c0 // BLK, world=nblk, nb=BLK)


rng = np.random.default_rng(7)
J = np.sort(rng.choice(n, 16, replace=False))
ax_res = -b_dev[:, :m].clone()                                  # A x - b
aj = torch.zeros((len(J), lda), dtype=torch.float64, device="cuda")
for c0 in range(0, n, BLK):
    w = min(BLK, n - c0)
    blk = a_block(c0, w)
    ax_res += x[:, c0:c0 + w] @ blk[:, :m]
    sel = (J >= c0) & (J < c0 + w)
    if sel.any():
        aj[torch.from_numpy(np.flatnonzero(sel)).cuda()] = blk[torch.from_numpy(J[sel] - c0).cuda()]
gram_a = torch.zeros((len(J), n), dtype=torch.float64, device="cuda")   # (A^T A)[:, J]^T
for c0 in range(0, n, BLK):
    w = min(BLK, n - c0)
    gram_a[:, c0:c0 + w] = aj[:, :m] @ a_block(c0, w)[:, :m].T
r_explicit = torch.linalg.norm(ax_res, dim=1)
out["resid_identity_max_rel"] = float((torch.abs(r_explicit - resid) / r_explicit).max())
# (R^T R)[:, J] from R streamed out of host memory by column blocks
rj = torch.zeros((len(J), n), dtype=torch.float64, device="cuda")     # R[:, J]^T
for i, j in enumerate(J):
    rj[i, :j + 1] = a_host[j, :j + 1].cuda()
gram_r = torch.zeros_like(gram_a)
for c0 in range(0, n, BLK):
    c1 = min(n, c0 + BLK)
    rb = a_host[c0:c1, :c1].cuda()                               # R[0:c1, c0:c1]^T (+ V below)
    rows = torch.arange(c1, device="cuda")[None, :]
    cols = torch.arange(c0, c1, device="cuda")[:, None]
    rb = torch.where(rows <= cols, rb, torch.zeros((), dtype=rb.dtype, device="cuda"))
    gram_r[:, c0:c1] = rj[:, :c1] @ rb.T
out["gram_cols"] = J.tolist()
out["gram_max_rel"] = float((gram_r - gram_a).abs().max() / gram_a.abs().max())
out["total_s"] = time.perf_counter() - t0
cudart.cudaHostUnregister(host_np.ctypes.data)
print(json.dumps(out), flush=True)
