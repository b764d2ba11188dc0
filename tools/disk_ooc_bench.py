"""Disk-staged QR on a generated config with an artificial HBM budget (development tool).

usage: python tools/disk_ooc_bench.py CFG BUDGET_GB TILE WORKDIR
Writes A as reference-format tiles under WORKDIR, factors it with DiskStagedQR
(host memory: a few pinned panel buffers), solves 64 slices, prints one JSON line.
Note: files written just before are usually still in the OS page cache, so the
"disk" read rate is an upper bound for a cold device."""
import json
import shutil
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.disk_ooc import DiskStagedQR  # noqa: E402
from paper_1907_01891_b200.tile_store import TiledMatrix  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
budget_gb = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tile = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
work = Path(sys.argv[4] if len(sys.argv) > 4 else "/tmp/qrb_disk")
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
x_true = cs.phantom_stack_device(cfg, 64)
bmat = x_true @ a_dev[:, :m]
b_dev = torch.zeros((64, lda), dtype=torch.float64, device="cuda")
b_dev[:, :m] = bmat
del a_dev, x_true
torch.cuda.empty_cache()
dst = TiledMatrix.create(m, n, tile, work / "factored")
q = DiskStagedQR(src, dst, budget_bytes=int(budget_gb * 2**30), io_threads=2)
st = q.factorize()
t0 = time.perf_counter()
x, r = q.solve(b_dev)
ts = time.perf_counter() - t0
q.close()
st.update({"cfg": cfg, "budget_gb": budget_gb, "tile": tile, "write_a_s": t_write_a,
           "solve64_s": ts, "resid_max": float(r.max()), "x_max": float(x.abs().max()),
           "read_GBps": st["read_bytes"] / max(st["read_s"], 1e-9) / 1e9,
           "write_GBps": st["write_bytes"] / max(st["write_s"], 1e-9) / 1e9})
print(json.dumps(st))
shutil.rmtree(work, ignore_errors=True)
