"""Graph-captured factorization (qrb_factorize for n <= graph_max_cols) and the
device-side CholeskyQR2 fallback it relies on.

The captured schedule must be the eager schedule: same kernels, same order, so
the factors are bitwise equal whether the factorization ran eagerly, was
captured, or was replayed -- also when a panel takes the Householder fallback
(chosen on the device by a flag, kernels.py:80-169 is the recurrence both
routes reproduce)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture
def nat():
    from paper_1907_01891_b200 import _native
    _native.load()
    saved = {k: _native.get_tuning(k) for k in ("graph_max_cols", "panel_algo", "cholqr_min_rows")}
    yield _native
    for k, v in saved.items():
        _native.set_tuning(k, v)


def _factor_runs(a, runs):
    from paper_1907_01891_b200.device import QrDevice
    m, n = a.shape
    out = []
    with QrDevice(m, n) as q:
        for _ in range(runs):
            q.set_matrix(a)
            q.factorize()
            out.append((q.get_matrix(), q.factors()))
    return out


def _same(x, y):
    np.testing.assert_array_equal(x[0], y[0])
    np.testing.assert_array_equal(x[1][0], y[1][0])
    np.testing.assert_array_equal(x[1][1], y[1][1])


def test_graph_replay_is_bitwise_the_eager_schedule(nat):
    from paper_1907_01891_b200 import ct_system as cs
    a = cs.dense_matrix(cs.config_geometry(1))          # config 1: 2160 x 1024
    nat.set_tuning("graph_max_cols", 0)
    eager = _factor_runs(a, 1)[0]
    nat.set_tuning("graph_max_cols", 16384)
    c0, r0 = nat.get_tuning("graph_captures"), nat.get_tuning("graph_replays")
    runs = _factor_runs(a, 4)                            # warm (eager), capture, 2 replays
    assert nat.get_tuning("graph_captures") == c0 + 1
    assert nat.get_tuning("graph_replays") == r0 + 2
    for r in runs:
        _same(r, eager)


def test_graph_replay_solves_like_the_oracle(nat):
    from conftest import rel_err, sign_normalise
    from oracle.tiled_qr import factorize_dense, solve_dense
    from paper_1907_01891_b200 import ct_system as cs
    from paper_1907_01891_b200.device import QrDevice
    nat.set_tuning("graph_max_cols", 16384)
    g = cs.config_geometry(1)
    a = cs.dense_matrix(g)
    b = cs.noisy_sinograms(a @ cs.phantom_stack(1, 4), 1)
    f = factorize_dense(a, 512, 128)
    x_ref = solve_dense(f, b)
    with QrDevice(*a.shape) as q:
        for _ in range(3):                               # the last one is a replay
            q.set_matrix(a)
            q.factorize()
        r = q.r_factor()
        x, resid, _ = q.solve(b)
    assert rel_err(sign_normalise(r), sign_normalise(np.triu(f.r()))) <= 1e-10
    assert rel_err(x, x_ref) <= 1e-8


def test_device_side_fallback_inside_the_graph(nat):
    """Zero and repeated columns make some CholeskyQR2 panels fall back; the
    predicated Householder kernels inside the captured graph give the same bits
    as the eager run and as the Householder-only schedule."""
    nat.set_tuning("cholqr_min_rows", 1024)
    nat.set_tuning("panel_algo", 0)
    rng = np.random.default_rng(5)
    m, n = 3000, 1024
    a = rng.standard_normal((m, n))
    a[:, 200] = 0.0
    a[:, 700] = a[:, 650]
    nat.set_tuning("graph_max_cols", 0)
    f0 = nat.get_tuning("cholqr_fallbacks")
    eager = _factor_runs(a, 1)[0]
    per_run = nat.get_tuning("cholqr_fallbacks") - f0
    assert per_run >= 2
    nat.set_tuning("graph_max_cols", 16384)
    f1 = nat.get_tuning("cholqr_fallbacks")
    runs = _factor_runs(a, 3)                            # eager warm, capture, replay
    assert nat.get_tuning("cholqr_fallbacks") - f1 == 3 * per_run
    for r in runs:
        _same(r, eager)
    tau = eager[1][0]
    assert tau[200] == 0.0


def test_tuning_change_recaptures(nat):
    from paper_1907_01891_b200 import ct_system as cs
    from paper_1907_01891_b200.device import QrDevice
    a = cs.dense_matrix(cs.config_geometry(0))
    nat.set_tuning("graph_max_cols", 16384)
    with QrDevice(*a.shape) as q:
        q.set_matrix(a)
        q.factorize()                                    # eager warm-up
        c0 = nat.get_tuning("graph_captures")
        q.set_matrix(a)
        q.factorize()
        ref = q.get_matrix()
        assert nat.get_tuning("graph_captures") == c0 + 1
        nat.set_tuning("graph_max_cols", 16384)          # any knob bumps the epoch
        q.set_matrix(a)
        q.factorize()
        assert nat.get_tuning("graph_captures") == c0 + 2
        np.testing.assert_array_equal(q.get_matrix(), ref)
