"""Disk-staged QR on a generated config with an HBM budget (run on the GPU box).

usage: python tools/disk_ooc_bench.py CFG BUDGET_GB TILE WORKDIR [uncached]
Writes A as reference-format tiles under WORKDIR, factors it with DiskStagedQR
(host memory: a few pinned panel buffers), solves 64 slices, prints one JSON line.
With "uncached" the OS page cache is dropped after A is written and the engine
runs with page_cache=False (reads from the device, writes synced and dropped):
the I/O rates are the device's, as on a host without RAM to spare for caching.
Checks: residual identity ||A x - b|| == ||(Q^T b)[n:m]|| against a device copy of
A kept only for checking, and recovery of the phantoms from noiseless sinograms.
"""
import json
import os
import shutil
import subprocess
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.disk_ooc import DiskStagedQR  # noqa: E402
from paper_1907_01891_b200.tile_store import TiledMatrix  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
budget_gb = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tile = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
work = Path(sys.argv[4] if len(sys.argv) > 4 else "/tmp/qrb_disk")
uncached = len(sys.argv) > 5 and sys.argv[5] == "uncached"
S = 64
shutil.rmtree(work, ignore_errors=True)
work.mkdir(parents=True)
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
a_dev = cs.densify_device(g, lda)
src = TiledMatrix.create(m, n, tile, work / "a")
t0 = time.perf_counter()
for c0 in range(0, n, 1024):
    w = min(1024, n - c0)
    src.write_columns(c0, w, a_dev[c0:c0 + w, :m].cpu().numpy().T)
t_write_a = time.perf_counter() - t0
dropped = False
if uncached:
    subprocess.run(["sync"], check=False)
    try:
        Path("/proc/sys/vm/drop_caches").write_text("3\n")
        dropped = True
    except OSError:
        pass
x_true = cs.phantom_stack_device(cfg, S)
ax = x_true @ a_dev[:, :m]
b_host = cs.noisy_sinograms(ax.cpu().numpy().T, cfg)
b_dev = torch.zeros((S, lda), dtype=torch.float64, device="cuda")
b_dev[:, :m] = torch.from_numpy(b_host.T.copy()).cuda()
dst = TiledMatrix.create(m, n, tile, work / "factored")
q = DiskStagedQR(src, dst, budget_bytes=int(budget_gb * 2**30), io_threads=2,
                 page_cache=not uncached)
clk = ClockSampler()
clk.start()
st = q.factorize()
clocks = clk.stop()
t0 = time.perf_counter()
x, r = q.solve(b_dev)
torch.cuda.synchronize()
ts = time.perf_counter() - t0
b0 = torch.zeros_like(b_dev)
b0[:, :m] = ax
x0, _ = q.solve(b0)
q.close()
r_explicit = torch.linalg.norm(x @ a_dev[:, :m] - b_dev[:, :m], dim=1)
st.update({"cfg": cfg, "m": m, "n": n, "a_gb": 8 * m * n / 1e9, "budget_gb": budget_gb,
           "tile": tile, "uncached": uncached, "page_cache_dropped": dropped,
           "write_a_s": t_write_a, "clocks": clocks,
           "solve64_s": ts, "slices_per_s": S / ts,
           "resid_identity_max_rel": float((torch.abs(r_explicit - r) / r_explicit).max()),
           "noiseless_x_rel_err": float((torch.linalg.norm(x0 - x_true, dim=1)
                                         / torch.linalg.norm(x_true, dim=1)).max()),
           "read_GBps": st["read_bytes"] / max(st["read_s"], 1e-9) / 1e9,
           "write_GBps": st["write_bytes"] / max(st["write_s"], 1e-9) / 1e9,
           "host_cores": len(os.sched_getaffinity(0))})
print(json.dumps(st))
shutil.rmtree(work, ignore_errors=True)
