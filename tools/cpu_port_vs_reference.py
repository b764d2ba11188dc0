"""Build-container check of the CPU baseline (not shipped, reads /root/reference):
per-task time of the six reference tile kernels -- the oracle port (what
bench.py's cpu_baseline / --impl reference legs time on the GPU box, where the
reference does not exist) against the REFERENCE package itself, numpy twin and
numba twin, on the same config-3 tiles (b = 2048, w = 128), and the config-3
extrapolation each gives.  Output: profiles/r02_cpu_port_vs_reference.json.

  NUMBA_CACHE_DIR=/tmp/numba python tools/cpu_port_vs_reference.py [reps]
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import bench  # noqa: E402
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402


def time_reference(kmod, t0, t1, b, w):
    out = {}
    a = t0.copy()
    tic = time.perf_counter()
    y, s_d = kmod.comp_dense_qr(a, w)
    out["comp_dense_qr"] = time.perf_counter() - tic
    t, d = y.copy(), t1.copy()
    tic = time.perf_counter()
    t, d, s_t = kmod.comp_td_qr(t, d, w)
    out["comp_td_qr"] = time.perf_counter() - tic
    c = t0.T.copy()
    tic = time.perf_counter()
    kmod.apply_left_qt_dense(y, s_d, c, w)
    out["apply_qt_dense"] = time.perf_counter() - tic
    f, g = t0.T.copy(), t1.T.copy()
    tic = time.perf_counter()
    kmod.apply_left_qt_td(d, s_t, f, g, w)
    out["apply_qt_td"] = time.perf_counter() - tic
    tic = time.perf_counter()
    kmod.gemm_nn_mo(f, t0, g)
    out["gemm_nn_mo"] = time.perf_counter() - tic
    rt = np.triu(t) + np.eye(b) * (np.abs(np.diag(t)).max() + 1.0)
    tic = time.perf_counter()
    kmod.trsm_lunn(rt, g, block=w)
    out["trsm_lunn"] = time.perf_counter() - tic
    return out


def med(runs):
    return {k: float(np.median([r[k] for r in runs])) for k in runs[0]}


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    from oocqr import kernels as K
    g = cs.config_geometry(3)
    m, n, S = g.n_rays, g.n_pixels, 256
    out = {"cores": len(os.sched_getaffinity(0)), "reps": reps, "workload": "config 3",
           "m": m, "n": n, "slices": S}
    for b in (1024, 2048, 4096):
        t0, t1 = bench.cpu_tiles(m, n, b, coo=cs.siddon_coo(g))
        w = 128
        port = med([bench.cpu_op_seconds(t0, t1, b, w) for _ in range(reps)])
        res = {"port": {"op_seconds": port, **_ex(bench.cpu_extrapolate(port, m, n, S, b))}}
        for path in ("numpy", "numba"):
            K.use_path(path)
            time_reference(K, t0, t1, b, w)              # warm-up (numba JIT)
            if path == "numba" and b > 2048:
                runs = [time_reference(K, t0, t1, b, w)]  # minutes per run
            else:
                runs = [time_reference(K, t0, t1, b, w) for _ in range(reps)]
            ref = med(runs)
            res["reference_" + path] = {"op_seconds": ref,
                                        **_ex(bench.cpu_extrapolate(ref, m, n, S, b))}
            res["port_over_reference_" + path] = {k: port[k] / ref[k] for k in port}
        out[f"b{b}"] = res
        print(json.dumps({f"b{b}": {k: v.get("qr_tflops") if isinstance(v, dict) else v
                                    for k, v in res.items()}}), flush=True)
    dst = ROOT / "profiles" / "r02_cpu_port_vs_reference.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(dst)


def _ex(e):
    return {"qr_tflops": e["qr_tflops"], "factor_s": e["factor_s"], "solve_s": e["solve_s"],
            "slices_per_s": e["slices_per_s"]}


if __name__ == "__main__":
    main()
