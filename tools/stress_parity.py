"""Randomised parity sweep (development tool): factorize + solve of random
shapes on the GPU against LAPACK (numpy), R up to row signs <= 1e-10, x <= 1e-8.

python tools/stress_parity.py [CASES] [SEED]
Shapes cover ragged panels (n not a multiple of 128 / 2), m barely above n,
short and tall panels on both panel routes, and graph-replayed repeats."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
worst_r = worst_x = 0.0
for it in range(cases):
    n = int(rng.choice([rng.integers(2, 130), rng.integers(130, 700), rng.integers(700, 2300)]))
    m = n + int(rng.choice([rng.integers(0, 8), rng.integers(8, 300), rng.integers(300, 4000)]))
    s = int(rng.integers(1, 9))
    a = rng.standard_normal((m, n))
    if rng.random() < 0.3:  # graded columns (cond ~1e4..1e6)
        a *= np.logspace(0, -rng.uniform(2, 5), n)
    b = rng.standard_normal((m, s))
    with QrDevice(m, n) as q:
        for rep in range(2 if rng.random() < 0.3 else 1):  # second pass replays the graph
            q.set_matrix(a)
            q.factorize()
            r = q.r_factor()
            x, res, _ = q.solve(b)
    r_ref = np.linalg.qr(a, mode="r")
    sg = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
    sg[sg == 0] = 1.0
    e_r = np.abs(r * sg[:, None] - r_ref).max() / np.abs(r_ref).max()
    x_ref = np.linalg.lstsq(a, b, rcond=None)[0]
    cond = np.linalg.cond(a)
    e_x = np.abs(x - x_ref).max() / np.abs(x_ref).max()
    res_ref = np.linalg.norm(a @ x_ref - b, axis=0)
    e_res = np.abs(res - res_ref).max() / max(res_ref.max(), 1e-300) if m > n else 0.0
    worst_r, worst_x = max(worst_r, e_r), max(worst_x, e_x / max(1.0, cond * 1e-4))
    ok = e_r <= 1e-10 and e_x <= 1e-8 * max(1.0, cond * 1e-4) and (e_res <= 1e-7 or res_ref.max() < 1e-9)
    if not ok or it % 20 == 0:
        print(f"{'ok ' if ok else 'BAD'} case {it}: {m} x {n}, {s} rhs, cond {cond:.1e}: "
              f"R {e_r:.1e} x {e_x:.1e} res {e_res:.1e}", flush=True)
    if not ok:
        sys.exit(1)
print(f"{cases} cases ok; worst R {worst_r:.1e}, worst x (cond-scaled) {worst_x:.1e}")
