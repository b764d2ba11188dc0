#!/usr/bin/env python
"""Benchmark of the hot path: fp64 blocked Householder QR of the CT system
matrix + multi-slice solve, on BASELINE.json's configuration 3 (256x256 image,
180 views x 384 bins -> A = 69120 x 65536 fp64, 36 GB; 256 noisy sinograms).

One step = reset A in HBM from its pristine copy (device-to-device), factor it
(qrb_factorize) and solve the slice batch against the new factors
(qrb_solve, device-resident B / X).  ``value`` is the QR TFLOP/s over the timed
steps (algorithmic 2mn^2 - 2n^3/3 flops / device time of the factorizations);
slices/s of the solve is reported beside it.  ``e2e`` repeats a step through
the public host-buffer API: pinned-host A and B copied in, X and the residual
norms copied out, all inside the timed region.

``--impl reference`` times the reference algorithm on the host cores, like for
like with our arm's workload: each of the reference's six tile kernels (the
oracle port of its numpy twin) on the workload's own b = 1024 tiles, the whole
QR and solve extrapolated as task count x seconds per task.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
For N > 1 launch under torchrun (one rank per GPU).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fp64 QR TFLOP/s (% of FP64 peak) at 1/2/4/8 GPUs; solved slices/sec"
UNIT = "TFLOP/s"
# measured FP64 tensor (DMMA.8x8x4) issue-rate peak of this pool's B200 at
# 1965 MHz, profiles/r01_fp64_pipe_probe.log (MEASURED_PEAKS.json has no fp64 entry)
FP64_PEAK_TFLOPS = 37.09
FP64_PEAK_SOURCE = "measured DMMA peak, profiles/r01_fp64_pipe_probe.log"
# the other two denominators SURVEY.md 8(d) asks for: nominal B200 FP64 tensor
# peak, and the measured cuBLAS DGEMM ceiling (torch.matmul fp64 8192^3,
# profiles/r01_fp64_pipe_probe.log)
FP64_NOMINAL_TFLOPS = 37.2
CUBLAS_DGEMM_TFLOPS = 35.47


def qr_flops(m: int, n: int) -> float:
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def solve_flops(m: int, n: int, s: int) -> float:
    return (4.0 * m * n - n * n) * s


# -- clocks sampler ---------------------------------------------------------------------


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int = 0):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# -- workload ------------------------------------------------------------------------------


def workload_config(cfg: int, m: int, n: int, slices: int, nb: int) -> dict:
    """The `config` object both arms report (same workload, same keys)."""
    return {"workload": f"config{cfg}: QR of A {m}x{n} fp64 + solve {slices} slices",
            "m": m, "n": n, "slices": slices, "panel_width": nb,
            "parallelism": "single GPU",
            "l2": ("inputs (A = %.1f GB) larger than L2 (126 MB)" % (m * n * 8 / 1e9))
                  if m * n * 8 > 126e6 else "inputs fit in L2 (small configuration)"}


def build_workload(cfg: int, slices: int | None, host_coo: bool = True):
    from paper_1907_01891_b200 import ct_system as cs
    g = cs.config_geometry(cfg)
    s = slices or cs.CONFIGS[cfg]["slices"]
    coo = cs.siddon_coo(g) if host_coo else None
    x_true = cs.phantom_stack(cfg, s)
    return g, coo, x_true, s


def densify_device(g, coo, lda: int):
    """Dense column-major A on the GPU (torch tensor (n, lda)) from host COO."""
    import torch
    r, c, v = coo
    a = torch.zeros((g.n_pixels, lda), dtype=torch.float64, device="cuda")
    flat = torch.from_numpy(c * lda + r).cuda()
    a.view(-1).index_put_((flat,), torch.from_numpy(v).cuda())
    return a


def measure_config(cfg: int, reps: int = 3) -> dict:
    """QR TFLOP/s and slices/s of another BASELINE configuration on this GPU
    (device-resident A and B, best of `reps` after a warm-up; reported beside
    the headline, not part of it)."""
    import torch
    from paper_1907_01891_b200 import ct_system as cs
    from paper_1907_01891_b200.device import QrDevice
    g = cs.config_geometry(cfg)
    m, n = g.n_rays, g.n_pixels
    S = cs.CONFIGS[cfg]["slices"]
    lda = (m + 31) // 32 * 32
    a = cs.densify_device(g, lda)
    xt = torch.from_numpy(np.ascontiguousarray(cs.phantom_stack(cfg, S).T)).cuda()   # (S, n)
    bh = cs.noisy_sinograms((xt @ a[:, :m]).cpu().numpy().T, cfg)                   # (m, S)
    b = torch.zeros((S, lda), dtype=torch.float64, device="cuda")
    b[:, :m] = torch.from_numpy(np.ascontiguousarray(bh.T)).cuda()
    x = torch.zeros((S, n + (n & 1)), dtype=torch.float64, device="cuda")
    q = QrDevice(m, n)
    fms, sms = [], []
    for it in range(reps + 1):
        q.set_matrix_device(a)
        f = q.factorize()["total_ms"]
        s_ = q.solve_device(b, x)["total_ms"]
        if it:
            fms.append(f)
            sms.append(s_)
    q.close()
    f_ms, s_ms = min(fms), min(sms)
    out = {"workload": f"config{cfg}: QR of A {m}x{n} + solve {S} slices", "m": m, "n": n,
           "slices": S, "qr_tflops": qr_flops(m, n) / (f_ms * 1e-3) / 1e12,
           "pct_fp64_peak": qr_flops(m, n) / (f_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
           "factor_ms": f_ms, "solve_ms": s_ms, "slices_per_s": S / (s_ms * 1e-3),
           "timing": f"best of {reps} after a warm-up, device-resident A and B",
           "pair_chain": [pair_chain_ms(m), pair_chain_ms(m - n + 256)]}
    del a, b, x, xt
    torch.cuda.empty_cache()
    return out


def pair_chain_ms(m: int, nb: int = 128, reps: int = 5) -> dict:
    """Latency of one panel-pair chain (factor panel a, Q_a^T on panel b, factor
    panel b, merge T2: qrb_op_panel_block on an m x 2nb block), the chain the
    look-ahead hides under the trailing update: on all SMs and with the GEMMs
    capped to the look-ahead's share (qrb tuning la_sms).  Best of `reps`."""
    import ctypes
    import torch
    from paper_1907_01891_b200 import _native as native
    lib = native.load()
    w = 2 * nb
    ld = m + (m & 1)
    g = torch.Generator(device="cuda").manual_seed(m)
    a0 = torch.randn((w, ld), dtype=torch.float64, device="cuda", generator=g)
    a = torch.empty_like(a0)
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    t = torch.zeros((2, nb, nb), dtype=torch.float64, device="cuda")
    t2 = torch.zeros((w, w), dtype=torch.float64, device="cuda")
    P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
    out = {"m": m, "w": w}
    la = native.get_tuning("la_sms")
    for label, cap in (("all_sms_ms", 0), (f"{la}_sms_ms", la)):
        native.set_tuning("grid_cap", cap)
        best = 1e30
        for it in range(reps + 1):
            a.copy_(a0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            native.check(lib.qrb_op_panel_block(P(a), ld, m, w, nb, P(tau), P(t), P(t2), w, None, 0),
                         "qrb_op_panel_block")
            e1.record()
            torch.cuda.synchronize()
            if it:
                best = min(best, e0.elapsed_time(e1))
        out[label] = round(best, 4)
    native.set_tuning("grid_cap", 0)
    return out


# -- CPU reference (oracle port of oocqr's numpy twin), extrapolated to the workload ----------

# reference tile size b: the fastest of b = 1024 / 2048 / 4096 for the reference's own
# numpy twin on config 3 (profiles/r02_cpu_port_vs_reference.json: 0.137 / 0.127 /
# 0.035 TFLOP/s extrapolated on 8 build cores; the port is within 10% per task)
CPU_TILE = 1024
CPU_INNER = 128      # reference inner block w (EngineConfig.inner_block default)


def task_counts(p: int, q: int, r: int) -> dict:
    """Tasks of the reference's left-looking tiled QR (task_engine.py:187-217) on a
    p x q tile grid and of its solve (:220-254) with r RHS block columns."""
    td = sum(p - 1 - k for k in range(q))
    return {"factor": {"comp_dense_qr": q, "comp_td_qr": td,
                       "apply_qt_dense": q * (q - 1) // 2,
                       "apply_qt_td": sum(p - 1 - j for k in range(q) for j in range(k))},
            "solve": {"apply_qt_dense": q * r, "apply_qt_td": td * r,
                      "gemm_nn_mo": q * (q - 1) // 2 * r, "trsm_lunn": q * r}}


def cpu_tiles(m: int, n: int, b: int, coo=None, a_cols=None):
    """Two b x b tiles of the workload's A (diagonal tile (0,0) and tile (1,0)),
    C-ordered like the reference's in-memory tiles (tile_store.py:193-194)."""
    if a_cols is None:
        r, c, v = coo
        sel = (c < b) & (r < 2 * b)
        a_cols = np.zeros((2 * b, b))
        a_cols[r[sel], c[sel]] = v[sel]
    blk = np.zeros((2 * b, b))
    blk[:a_cols.shape[0], :a_cols.shape[1]] = a_cols[:2 * b, :b]
    return np.ascontiguousarray(blk[:b]), np.ascontiguousarray(blk[b:])


def cpu_op_seconds(t0: np.ndarray, t1: np.ndarray, b: int, w: int) -> dict:
    """One timed execution of each reference tile kernel (oracle port of the
    numpy twin, kernels.py:296-455) on the workload's own tiles.  The applies
    reuse the factors the QRs just produced (the reference's data flow)."""
    from oracle import tiled_qr as orc
    out = {}
    a = t0.copy()
    tic = time.perf_counter()
    y, s_d = orc.comp_dense_qr(a, w)
    out["comp_dense_qr"] = time.perf_counter() - tic
    t, d = y.copy(), t1.copy()
    tic = time.perf_counter()
    t, d, s_t = orc.comp_td_qr(t, d, w)
    out["comp_td_qr"] = time.perf_counter() - tic
    c = t0.T.copy()                                      # a b x b tile to update
    tic = time.perf_counter()
    orc.apply_left_qt_dense(y, s_d, c, w)
    out["apply_qt_dense"] = time.perf_counter() - tic
    f, g = t0.T.copy(), t1.T.copy()
    tic = time.perf_counter()
    orc.apply_left_qt_td(d, s_t, f, g, w)
    out["apply_qt_td"] = time.perf_counter() - tic
    tic = time.perf_counter()
    orc.gemm_nn_mo(f, t0, g)
    out["gemm_nn_mo"] = time.perf_counter() - tic
    rt = np.triu(t) + np.eye(b) * (np.abs(np.diag(t)).max() + 1.0)   # well-posed triangle
    tic = time.perf_counter()
    orc.trsm_lunn(rt, g, block=w)
    out["trsm_lunn"] = time.perf_counter() - tic
    return out


def cpu_extrapolate(op_s: dict, m: int, n: int, slices: int, b: int) -> dict:
    """Reference time of the whole workload = sum over ops of (task count x
    measured seconds per task) -- tiles are always full b x b (zero padded,
    tile_store.py:186-187), so every task of a kind costs the same."""
    p, q, r = -(-m // b), -(-n // b), -(-slices // b)
    cnt = task_counts(p, q, r)
    f_s = sum(cnt["factor"][k] * op_s[k] for k in cnt["factor"])
    s_s = sum(cnt["solve"][k] * op_s[k] for k in cnt["solve"])
    return {"factor_s": f_s, "solve_s": s_s, "grid": [p, q, r], "task_counts": cnt,
            "qr_tflops": qr_flops(m, n) / f_s / 1e12, "slices_per_s": slices / s_s}


def cpu_baseline_run(m: int, n: int, slices: int, coo=None, a_cols=None, steps: int = 1,
                     warmup: int = 0, b: int = CPU_TILE, w: int = CPU_INNER,
                     min_seconds: float = 0.0) -> dict:
    """steps timed executions of the six tile kernels -- more, up to 200, until
    min_seconds of CPU work have been sampled (the bench's cpu_baseline: ~10 s)."""
    t0, t1 = cpu_tiles(m, n, b, coo, a_cols)
    for _ in range(warmup):
        cpu_op_seconds(t0, t1, b, w)
    runs, wall = [], []
    while len(runs) < steps or (sum(wall) < min_seconds and len(runs) < 200):
        tic = time.perf_counter()
        runs.append(cpu_op_seconds(t0, t1, b, w))
        wall.append(time.perf_counter() - tic)
    steps = len(runs)
    op_s = {k: float(np.median([r_[k] for r_ in runs])) for k in runs[0]}
    ex = cpu_extrapolate(op_s, m, n, slices, b)
    ex.update({"op_seconds": op_s, "sample_s_per_step": float(np.mean(wall)), "tile": b,
               "inner_block": w, "cores": len(os.sched_getaffinity(0)),
               "sample": (f"oracle port of oocqr's numpy twin (OOCQR_DISABLE_NUMBA=1 path): one "
                          f"execution of each of the 6 tile kernels on the workload's own b={b} "
                          f"tiles (w={w}) per step, median over {steps} steps "
                          f"({sum(wall):.1f} s sampled); the {m}x{n} QR and "
                          f"the {slices}-slice solve EXTRAPOLATED as task count x time per task "
                          f"(grid {-(-m // b)}x{-(-n // b)}, tile I/O excluded, which favours the "
                          f"reference)")})
    return ex


def reference_arm(args, rank: int):
    if rank != 0:
        return
    from paper_1907_01891_b200 import ct_system as cs
    g = cs.config_geometry(args.config)
    m, n = g.n_rays, g.n_pixels
    S = args.slices or cs.CONFIGS[args.config]["slices"]
    b = min(CPU_TILE, n)
    # the two b x b tiles of A the sample runs on: Siddon rays of the first 2b rows
    r0, c0, v0 = cs.siddon_coo(g)
    coo = (r0, c0, v0)
    ex = cpu_baseline_run(m, n, S, coo=coo, steps=args.steps, warmup=args.warmup, b=b)
    val = ex["qr_tflops"]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ex["sample_s_per_step"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Siddon fan-beam A, seeded)",
        "config": workload_config(args.config, m, n, S, args.nb),
        "extrapolated": True,
        "reference_factor_s": ex["factor_s"], "reference_solve_s": ex["solve_s"],
        "slices_per_s": ex["slices_per_s"], "op_seconds": ex["op_seconds"],
        "task_counts": ex["task_counts"],
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": ex["cores"], "kind": "port",
                         "sample": ex["sample"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# -- our arm -----------------------------------------------------------------------------------


def ours_arm(args, rank: int, world: int):
    import torch
    from paper_1907_01891_b200 import _native as native
    from paper_1907_01891_b200 import ct_system as cs
    from paper_1907_01891_b200.device import QrDevice, launch_count

    if world > 1 or args.force_dist:
        from paper_1907_01891_b200 import dist
        return dist.bench_rank(args, rank, world)

    torch.cuda.set_device(0)
    t_setup = time.perf_counter()
    g, _, x_true, S = build_workload(args.config, args.slices, host_coo=False)
    m, n = g.n_rays, g.n_pixels
    lda = (m + 31) // 32 * 32
    a_dev = cs.densify_device(g, lda)          # sm_100a Siddon kernel, straight into HBM
    torch.cuda.synchronize()
    densify_s = time.perf_counter() - t_setup
    cpu_cols = a_dev[:min(CPU_TILE, n), :min(2 * CPU_TILE, m)].cpu().numpy().T.copy()
    # sinograms b = A x + 1% noise (seeded per slice); A x via the device matrix
    xt = torch.from_numpy(np.ascontiguousarray(x_true.T)).cuda()        # (S, n)
    ax_dev = xt @ a_dev[:, :m]                                           # (S, m), noiseless
    ax = ax_dev.cpu().numpy().T                                          # (m, S)
    b_host = cs.noisy_sinograms(ax, args.config)
    ldb = lda
    b_dev = torch.zeros((S, ldb), dtype=torch.float64, device="cuda")
    b_dev[:, :m] = torch.from_numpy(np.ascontiguousarray(b_host.T)).cuda()
    x_dev = torch.zeros((S, (n + 1) // 2 * 2), dtype=torch.float64, device="cuda")
    r_dev = torch.zeros(S, dtype=torch.float64, device="cuda")
    del xt
    q = QrDevice(m, n, args.nb)
    q.set_profiling(True)
    setup_s = time.perf_counter() - t_setup

    def step():
        q.set_matrix_device(a_dev)
        frep = q.factorize()
        srep = q.solve_device(b_dev, x_dev, r_dev)
        return frep, srep

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    launches0 = launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    freps, sreps = [], []
    for _ in range(args.steps):
        fr, sr = step()
        freps.append(fr)
        sreps.append(sr)
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = launch_count() - launches0
    step_ms = e0.elapsed_time(e1) / args.steps
    f_ms = float(np.mean([r["total_ms"] for r in freps]))
    s_ms = float(np.mean([r["total_ms"] for r in sreps]))
    fl = qr_flops(m, n)
    value = fl / (f_ms * 1e-3) / 1e12
    slices_per_s = S / (s_ms * 1e-3)

    # dominant kernel roofline from the live CUDA-event kernel accounting
    kstats: dict = {}
    for rep in freps + sreps:
        for name, k in rep["kernels"].items():
            acc = kstats.setdefault(name, {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
            for key in acc:
                acc[key] += k[key]
    # the dominant kernel by total device time: the trailing-update NN GEMM
    # (gemm_nn_sub_asyncepi) counts its full-grid launches AND the capped ones
    # that run beside the look-ahead panel (the same kernel on 148 - la_sms CTAs)
    zero = {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0}
    fam = {"gemm_tn": dict(kstats.get("gemm_tn", zero)), "gemm_nn": dict(kstats.get("gemm_nn", zero))}
    for key in fam["gemm_nn"]:
        fam["gemm_nn"][key] += kstats.get("gemm_nn_capped", zero)[key]
    dom = max(fam, key=lambda k: fam[k]["ms"])
    dk = fam[dom]
    achieved = dk["flops"] / (dk["ms"] * 1e-3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": UNIT,
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None, "kernel": dom,
                "kernel_name": {"gemm_nn": "gemm_nn_sub_asyncepi (C -= V W2, full-grid + capped "
                                           "launches)",
                                "gemm_tn": "gemm_dmma_kernel<KMAJOR=1> (W = V^T C)"}[dom],
                "peak_source": FP64_PEAK_SOURCE,
                "per_launch_flops": dk["flops"] / dk["launches"],
                "avg_launch_ms": dk["ms"] / dk["launches"],
                "time_share": {k: round(v["ms"] / sum(x["ms"] for x in kstats.values()), 4)
                               for k, v in fam.items()}}
    roofline.update(_ncu_traffic(dom, m, n, args.nb))
    if "gemm_nn_capped" in kstats and kstats["gemm_nn_capped"]["launches"]:
        ck, uk = kstats["gemm_nn_capped"], kstats["gemm_nn"]
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        la_sms = native.get_tuning("la_sms")
        if m >= native.get_tuning("la_tall_rows"):
            # tall steps (>= la_tall_rows rows: nearly all of the capped time at this
            # size) leave the chain la_sms_tall SMs
            la_sms = max(la_sms, native.get_tuning("la_sms_tall"))
        ca = ck["flops"] / (ck["ms"] * 1e-3) / 1e12
        ua = uk["flops"] / (uk["ms"] * 1e-3) / 1e12
        # NN's two launch kinds: whole-GPU rate of the full-grid launches, and the
        # capped launches' rate per SM they were given (148 - la_sms CTAs while the
        # next panel pair is factored on the other SMs)
        roofline["nn_parts"] = {
            "full_grid": {"achieved": ua, "frac": ua / FP64_PEAK_TFLOPS,
                          "launches": uk["launches"], "ms": uk["ms"]},
            # (chain-bound late steps leave the chain up to la_sms_max SMs, so a few
            # capped launches had fewer SMs than this: frac_of_its_sms is a lower bound)
            "capped": {"achieved": ca, "sms": sms - la_sms,
                       "sms_min": sms - max(la_sms, native.get_tuning("la_sms_max")),
                       "frac_of_its_sms": ca / (FP64_PEAK_TFLOPS * (sms - la_sms) / sms),
                       "launches": ck["launches"], "ms": ck["ms"]}}
    shares = {k: round(v["ms"] / sum(x["ms"] for x in kstats.values()), 4) for k, v in kstats.items()}
    roofline["kernel_tflops"] = {k: round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 3)
                                 for k, v in kstats.items() if v["ms"] > 0 and k.startswith("gemm")}

    # residual sanity of the last step: GPU residual identity vs explicit ||Ax - b||
    x_last = x_dev[:, :n]
    r_explicit = torch.linalg.norm(x_last @ a_dev[:, :m] - b_dev[:, :m], dim=1)
    resid_rel = float((torch.abs(r_explicit - r_dev) / r_explicit).max())
    resid_dbg = {"explicit": r_explicit[:3].tolist(), "identity": r_dev[:3].tolist(),
                 "x_absmax": float(x_last.abs().max())}
    # image quality of the reconstructed slices vs the phantoms (paper Tables IV/V metrics)
    from paper_1907_01891_b200 import metrics
    xt_dev = torch.from_numpy(x_true).cuda()
    quality = {"psnr_avg_db": float(metrics.psnr(xt_dev, x_last.T, g.image_pixels).mean()),
               "ssim_avg": float(metrics.ssim(xt_dev, x_last.T, g.image_pixels).mean()),
               "relative_residual": metrics.relative_residual(a_dev, x_last.T, b_dev[:, :m].T, m),
               "note": "noisy sinograms (1% Gaussian), least-squares solution"}
    # the same slices from the noiseless sinograms A x_true: the least-squares
    # solution must reproduce the phantoms (size-independent correctness check;
    # the noisy numbers above measure the conditioning of A, not the solver)
    b0 = torch.zeros_like(b_dev)
    b0[:, :m] = ax_dev
    x0 = torch.zeros_like(x_dev)
    q.solve_device(b0, x0, None)
    x0n = x0[:, :n]
    err = torch.linalg.norm(x0n - xt_dev.T, dim=1) / torch.linalg.norm(xt_dev.T, dim=1)
    quality["noiseless"] = {"psnr_avg_db": float(metrics.psnr(xt_dev, x0n.T, g.image_pixels).mean()),
                            "x_rel_err_max": float(err.max())}
    del xt_dev, b0, x0, ax_dev

    # config 5: solve throughput of a 4096-slice batch against the config-3 factors
    cfg5 = None
    if args.config == 3 and args.cfg5_slices > 0:
        S5 = args.cfg5_slices
        x5 = cs.phantom_stack_device(5, S5)                                   # (S5, n)
        ax5 = (x5 @ a_dev[:, :m]).cpu().numpy().T                             # (m, S5)
        del x5
        b5 = torch.zeros((S5, ldb), dtype=torch.float64, device="cuda")
        b5[:, :m] = torch.from_numpy(np.ascontiguousarray(cs.noisy_sinograms(ax5, 5).T)).cuda()
        del ax5
        x5o = torch.zeros((S5, (n + 1) // 2 * 2), dtype=torch.float64, device="cuda")
        r5 = torch.zeros(S5, dtype=torch.float64, device="cuda")
        q.solve_device(b5, x5o, r5)                                           # warm-up
        reps5 = [q.solve_device(b5, x5o, r5) for _ in range(2)]
        s5_ms = float(np.mean([r["total_ms"] for r in reps5]))
        cfg5 = {"workload": f"config5: solve {S5} slices on the config-3 factors",
                "slices": S5, "solve_ms": s5_ms, "slices_per_s": S5 / (s5_ms * 1e-3),
                "solve_tflops": solve_flops(m, n, S5) / (s5_ms * 1e-3) / 1e12}
        del b5, x5o, r5
        torch.cuda.empty_cache()

    # end-to-end through the public host API (pinned host A and B, host X out)
    # exact-size page-locked host A (torch's pinned allocator rounds up to a power of two)
    from paper_1907_01891_b200.device import PinnedHostArray
    a_pin_hold = PinnedHostArray((n, lda))
    a_pin = torch.from_numpy(a_pin_hold.array)
    a_pin.copy_(a_dev)
    b_pin = torch.empty((S, ldb), dtype=torch.float64, pin_memory=True)
    b_pin.copy_(b_dev)
    x_pin = torch.empty((S, n), dtype=torch.float64, pin_memory=True)
    a_view = a_pin.numpy().T[:m, :]          # m x n column-major view, ld = lda
    b_view = b_pin.numpy().T[:m, :]
    x_view = x_pin.numpy().T                 # n x S column-major
    del a_dev
    torch.cuda.empty_cache()
    q.set_profiling(False)
    e2e_steps = max(1, args.e2e_steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(e2e_steps):
        frep_e2e = q.factorize_host(a_view)      # chunked H2D overlapped with the QR
        _, resid_host, _ = q.solve(b_view, out=x_view)
    e3.record()
    torch.cuda.synchronize()
    e2e_s = max(e2.elapsed_time(e3) * 1e-3, 0.0) / e2e_steps
    wall_e2e = (time.perf_counter() - t0) / e2e_steps
    e2e = {"value": fl / e2e_s / 1e12, "unit": UNIT,
           "h2d_bytes_per_step": int(m * n * 8 + m * S * 8),
           "d2h_bytes_per_step": int(n * S * 8 + S * 8),
           "ms_per_step": e2e_s * 1e3, "wall_ms_per_step": wall_e2e * 1e3,
           "slices_per_s": S / e2e_s,
           "h2d_ms_overlapped": frep_e2e["h2d_ms"],
           "path": "QrDevice.factorize_host(pinned host A; chunked H2D overlapped with the "
                   "left-looking chunk order) + solve(host B -> host X)"}
    # the host-API result against the device-path result of the timed steps (the
    # two factorizations run the columns in a different order: rounding only)
    xd = x_dev[:, :n].cpu().numpy().T
    rd = r_dev.cpu().numpy()
    e2e["check"] = {"x_max_rel_vs_device_path": float(np.abs(x_view - xd).max() / np.abs(xd).max()),
                    "resid_max_rel_vs_device_path":
                        float((np.abs(np.asarray(resid_host) - rd) / np.abs(rd)).max())}
    del xd, rd
    q.close()
    del a_pin, b_pin, x_pin
    a_pin_hold.close()
    others = {}
    if args.config == 3 and args.other_configs:
        for c in (1, 2):
            others[f"config{c}"] = measure_config(c)

    cpu = cpu_baseline_run(m, n, S, a_cols=cpu_cols, steps=5, warmup=1, b=min(CPU_TILE, n),
                           min_seconds=10.0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Siddon fan-beam A from seeded geometry; seeded 10-ellipse phantoms, "
                "1% Gaussian noise)",
        "config": workload_config(args.config, m, n, S, args.nb),
        "pct_fp64_peak": value / FP64_PEAK_TFLOPS,
        "pct_fp64_nominal": value / FP64_NOMINAL_TFLOPS,
        "vs_cublas_dgemm": value / CUBLAS_DGEMM_TFLOPS,
        "slices_per_s": slices_per_s,
        "solve_tflops": solve_flops(m, n, S) / (s_ms * 1e-3) / 1e12,
        "factor_ms": f_ms, "solve_ms": s_ms,
        "roofline": roofline, "kernel_time_share": shares,
        "cpu_baseline": {"value": cpu["qr_tflops"], "unit": UNIT, "cores": cpu["cores"],
                         "kind": "port", "sample": cpu["sample"], "extrapolated": True,
                         "factor_s": cpu["factor_s"], "solve_s": cpu["solve_s"],
                         "slices_per_s": cpu["slices_per_s"], "op_seconds": cpu["op_seconds"]},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "config5": cfg5, "other_configs": others or None, "quality": quality,
        "pair_chain": [pair_chain_ms(m, args.nb), pair_chain_ms(m - n + 2 * args.nb, args.nb)],
        "check": {"resid_identity_max_rel": resid_rel, "resid_sample": resid_dbg},
        "setup_s": setup_s, "densify_s": densify_s,
    }
    emit(line)


def claim_stdout() -> None:
    """Keep fd 1 for the one JSON line; anything native libraries write to fd 1
    (e.g. the NCCL version banner) goes to stderr instead.  The saved fd is kept
    in the environment because dist.py re-imports this file as `bench`."""
    if "QRB_JSON_FD" not in os.environ:
        sys.stdout.flush()
        os.environ["QRB_JSON_FD"] = str(os.dup(1))
        os.dup2(2, 1)


def emit(line: dict) -> None:
    sys.stdout.flush()
    os.write(int(os.environ.get("QRB_JSON_FD", "1")), (json.dumps(line) + "\n").encode())


def _ncu_traffic(kernel: str, m: int, n: int, nb: int) -> dict:
    """DRAM bytes of one launch of the dominant kernel from the committed `ncu
    --set full` captures of the config-3 bench (the longest launch of the first
    pair step; its shape in the launch_shape line):
      gemm_nn: profiles/r01_ncu_full_gemm_nn_k512_config3.txt (C -= V W2)
      gemm_tn: profiles/r01_ncu_full_gemm_tn_k512_config3.txt (W = V^T C)
    (the first steps use 4-panel blocks; K = 256 captures of the pair steps are
    kept beside them as *_k256_*).
    Read from the committed summaries, not measured in this run."""
    name = {"gemm_nn": "r01_ncu_full_gemm_nn_k512_config3.txt",
            "gemm_tn": "r01_ncu_full_gemm_tn_k512_config3.txt"}.get(kernel)
    prof = Path(__file__).resolve().parent / "profiles" / (name or "-")
    if name is None or (m, n) != (69120, 65536) or not prof.is_file():
        return {}
    vals, shape = {}, None
    for line in prof.read_text().splitlines():
        parts = line.split(",")
        if len(parts) >= 2 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            unit = parts[2].strip().lower() if len(parts) > 2 else "gbyte"
            vals[parts[0]] = float(parts[1]) * (1e6 if unit.startswith("m") else 1e9)
        if parts[0] in ("launch_shape", "launch_shape_tn"):
            shape = (parts[0], tuple(int(x) for x in parts[1:4]))
    if len(vals) != 2 or shape is None:
        return {}
    kind, (d0, d1, d2) = shape
    if kind == "launch_shape":        # NN: C (d0 x d1) read + write, V (d0 x d2), W2 (d2 x d1)
        algo = 8.0 * (2 * d0 * d1 + d0 * d2 + d2 * d1)
    else:                             # TN: W (d0 x d1) = V^T C, V (d2 x d0), C (d2 x d1)
        algo = 8.0 * (d2 * d1 + d2 * d0 + d0 * d1)
    return {"traffic": sum(vals.values()), "traffic_unit": "bytes",
            "traffic_launch": f"one launch {d0}x{d1}x{d2} (ncu --set full, profiles/{name})",
            "traffic_algorithmic": algo}


def relaunch_under_torchrun(n: int) -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    env = {k: v for k, v in os.environ.items() if k != "QRB_JSON_FD"}
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--slices", type=int, default=None)
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cfg5-slices", type=int, default=4096,
                    help="slices of the config-5 solve-throughput run (0 = skip)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--other-configs", type=int, default=1,
                    help="with config 3: also report configs 1 and 2 on this GPU (1) or not (0)")
    ap.add_argument("--lean-solve", action="store_true",
                    help="multi-GPU: stream V and R instead of replicating the factors")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: functional check of the multi-rank path with ranks sharing one GPU")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU (torch.distributed) path even at N=1")
    args = ap.parse_args()
    if args.gpus > 1 and args.impl == "ours" and args.dist_backend == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            # one rank per GPU over NCCL: fail before starting ranks that cannot get a device
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs on this node, found {have} "
                  "(--dist-backend gloo runs the multi-rank path with ranks sharing a GPU)",
                  file=sys.stderr)
            sys.exit(2)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start N ranks (one per
        # GPU) under torch.distributed.run on this node; rank 0 prints the line
        sys.exit(relaunch_under_torchrun(args.gpus))
    claim_stdout()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    ours_arm(args, rank, world)


if __name__ == "__main__":
    main()
