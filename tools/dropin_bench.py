"""The reference-facing drop-in API at scale (run on the GPU box):

    python tools/dropin_bench.py CFG TILE WORKDIR [uncached]

Writes A and the sinogram stack B of configuration CFG as reference-format tile
stores under WORKDIR, then runs ``paper_1907_01891_b200.factorize`` and
``solve`` exactly as a caller of ``oocqr.factorize`` / ``solve`` would
(task_engine.py:606-685) and prints their RunReports and wall times as one JSON
line.  With "uncached" the OS page cache is dropped after the stores are
written, so the tile reads come from the device.
"""
import json
import shutil
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1907_01891_b200 as pkg  # noqa: E402
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
work = Path(sys.argv[3] if len(sys.argv) > 3 else "/tmp/qrb_dropin")
uncached = len(sys.argv) > 4 and sys.argv[4] == "uncached"
shutil.rmtree(work, ignore_errors=True)
work.mkdir(parents=True)
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
S = cs.CONFIGS[cfg]["slices"]
lda = (m + 31) // 32 * 32
a_dev = cs.densify_device(g, lda)
am = pkg.TiledMatrix.create(m, n, tile, work / "a")
for c0 in range(0, n, 2048):
    w = min(2048, n - c0)
    am.write_columns(c0, w, a_dev[c0:c0 + w, :m].cpu().numpy().T)
x_true = cs.phantom_stack_device(cfg, S)
bh = cs.noisy_sinograms((x_true @ a_dev[:, :m]).cpu().numpy().T, cfg)   # (m, S)
del a_dev
torch.cuda.empty_cache()
bm = pkg.TiledMatrix.create(m, S, tile, work / "b")
bm.write_columns(0, S, np.asfortranarray(bh))
dropped = False
if uncached:
    subprocess.run(["sync"], check=False)
    try:
        Path("/proc/sys/vm/drop_caches").write_text("3\n")
        dropped = True
    except OSError:
        pass
conf = pkg.EngineConfig(tile_size=tile, inner_block=128)
t0 = time.perf_counter()
factors, frep = pkg.factorize(am, conf, work / "f")
t_f = time.perf_counter() - t0
t0 = time.perf_counter()
xm, srep = pkg.solve(factors, bm, conf, work / "out")
t_s = time.perf_counter() - t0
x = pkg.gather_matrix(xm)
fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def rep_dict(r):
    return {k: getattr(r, k) for k in ("total_seconds", "compute_seconds", "io_read_seconds",
                                        "io_write_seconds", "h2d_seconds", "tiles_read",
                                        "tiles_written", "task_count")}


out = {"cfg": cfg, "m": m, "n": n, "slices": S, "tile": tile, "uncached": uncached,
       "page_cache_dropped": dropped, "factorize_wall_s": t_f, "solve_wall_s": t_s,
       "qr_tflops_wall": fl / t_f / 1e12, "qr_tflops_device": frep.gpu_tflops,
       "factorize_report": rep_dict(frep), "solve_report": rep_dict(srep),
       "x_absmax": float(np.abs(x).max())}
print(json.dumps(out), flush=True)
shutil.rmtree(work, ignore_errors=True)
