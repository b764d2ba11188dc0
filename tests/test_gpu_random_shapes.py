"""Randomised shapes through the drop-in device path against LAPACK (numpy):
ragged panel counts, m barely above n, short and tall panels (both panel
routes), graded columns, graph-replayed repeats.  north_star tolerances: R up
to row signs <= 1e-10, x <= 1e-8 (scaled by cond beyond 1e4), residual norms.
`tools/stress_parity.py` runs the same sweep with more cases."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_random_shapes_match_lapack(seed):
    from paper_1907_01891_b200.device import QrDevice

    rng = np.random.default_rng(seed)
    for _ in range(14):
        n = int(rng.choice([rng.integers(2, 130), rng.integers(130, 700), rng.integers(700, 2300)]))
        m = n + int(rng.choice([rng.integers(0, 8), rng.integers(8, 300), rng.integers(300, 4000)]))
        s = int(rng.integers(1, 9))
        a = rng.standard_normal((m, n))
        if rng.random() < 0.3:
            a *= np.logspace(0, -rng.uniform(2, 5), n)
        b = rng.standard_normal((m, s))
        with QrDevice(m, n) as q:
            for _rep in range(2 if rng.random() < 0.3 else 1):  # the second pass replays the graph
                q.set_matrix(a)
                q.factorize()
                r = q.r_factor()
                x, res, _ = q.solve(b)
        r_ref = np.linalg.qr(a, mode="r")
        sg = np.sign(np.diag(r)) * np.sign(np.diag(r_ref))
        sg[sg == 0] = 1.0
        assert np.abs(r * sg[:, None] - r_ref).max() <= 1e-10 * np.abs(r_ref).max(), (m, n)
        x_ref = np.linalg.lstsq(a, b, rcond=None)[0]
        cond = np.linalg.cond(a)
        assert np.abs(x - x_ref).max() <= 1e-8 * max(1.0, cond * 1e-4) * np.abs(x_ref).max(), (m, n)
        res_ref = np.linalg.norm(a @ x_ref - b, axis=0)
        if m > n and res_ref.max() > 1e-9:
            np.testing.assert_allclose(res, res_ref, rtol=1e-7, err_msg=str((m, n)))
