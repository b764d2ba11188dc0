"""Timeline of one factorization of a small configuration (development tool).

python tools/small_cfg_trace.py CFG [REPS]
Prints the best factor time over REPS, then a CUPTI kernel timeline (torch
profiler) of one more factorization: busy time, idle gaps between kernels, and
the kernels by total time.  Used to see where configs 1-2 lose to launch gaps.
"""
import json
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_1907_01891_b200 import ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
lda = (m + 31) // 32 * 32
a = cs.densify_device(g, lda)
q = QrDevice(m, n)
fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3
best = 1e30
for it in range(reps + 1):
    q.set_matrix_device(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = q.factorize()
    wall = (time.perf_counter() - t0) * 1e3
    if it:
        best = min(best, rep["total_ms"])
    print(f"rep {it}: total_ms {rep['total_ms']:.3f} wall {wall:.3f} launches "
          f"{rep.get('kernel_launches')}")
print(json.dumps({"cfg": cfg, "m": m, "n": n, "best_ms": best, "tflops": fl / best / 1e9}))

q.set_profiling(True)
q.set_matrix_device(a)
rep = q.factorize()
q.set_profiling(False)
for k, v in rep.get("kernels", {}).items():
    print(f"kind {k:15s} {v['ms']:9.2f} ms {v['launches']:6d} scopes "
          f"{v['flops'] / max(v['ms'], 1e-9) / 1e9:7.2f} TFLOP/s")

from torch.profiler import ProfilerActivity, profile  # noqa: E402

q.set_matrix_device(a)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    q.factorize()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = sorted(ev, key=lambda e: e.time_range.start)
kern = [e for e in ev if "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
t_start, t_end = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy, last_end, gaps = 0.0, t_start, []
per = defaultdict(lambda: [0, 0.0])
for e in ev:
    s, f = e.time_range.start, e.time_range.end
    if s > last_end:
        gaps.append((s - last_end, e.name[:60]))
    busy += max(0.0, f - max(s, last_end))
    last_end = max(last_end, f)
    per[e.name[:70]][0] += 1
    per[e.name[:70]][1] += f - s
span = t_end - t_start
print(f"span {span:.1f} us, busy {busy:.1f} us ({100 * busy / span:.1f}%), events {len(ev)} "
      f"(kernels {len(kern)}), gaps {len(gaps)} total {sum(g_ for g_, _ in gaps):.1f} us")
for name, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {t:9.1f} us  {c:5d}x  {name}")
gaps.sort(reverse=True)
print("largest gaps (us, before kernel):")
for g_, nm in gaps[:15]:
    print(f"  {g_:8.1f}  {nm}")
q.close()
