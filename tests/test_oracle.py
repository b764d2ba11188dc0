"""The CPU oracle (numpy restatement of the reference) pinned against golden
vectors produced by running the reference itself (tests/golden/make_golden.py)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, rel_err, sign_normalise
from oracle import tiled_qr as orc
from paper_1907_01891_b200 import ct_system as cs

KAT = json.loads((GOLDEN / "ref_meta.json").read_text())["kat"]


# -- known-answer vectors (reference kernels) ------------------------------------------


def test_kat_dense_two_vector_column():
    a = np.zeros((4, 4))
    a[0, 0], a[1, 0] = 3.0, 4.0
    a, _ = orc.comp_dense_qr(a, 2)
    assert abs(a[0, 0]) == pytest.approx(KAT["dense_3_4_r00"], rel=1e-15)


def test_kat_td_scalar_pair():
    t, _, _ = orc.comp_td_qr(np.array([[1.0]]), np.array([[1.0]]), 1)
    assert abs(t[0, 0]) == pytest.approx(KAT["td_1_1_r00"], rel=1e-15)


def test_kat_trsm_and_singular_columns():
    x = orc.trsm_lunn(np.array([[2.0, 1.0], [0.0, 4.0]]), np.array([[5.0], [8.0]]))
    np.testing.assert_allclose(x[:, 0], KAT["trsm_2x2"], rtol=1e-15)
    rt = np.eye(4)
    rt[2, 2] = 0.0
    with pytest.raises(orc.OracleSingularError) as e:
        orc.trsm_lunn(rt, np.ones((4, 1)), col_offset=12)
    assert e.value.global_column == KAT["trsm_singular_col"]
    rt = np.eye(3)
    rt[1, 1] = 1e-308
    with pytest.raises(orc.OracleSingularError) as e:
        orc.trsm_lunn(rt, np.ones((3, 1)))
    assert e.value.global_column == KAT["trsm_subthreshold_col"]


def test_identity_tile_gives_zero_reflectors():
    a, s = orc.comp_dense_qr(np.eye(6), 2)
    np.testing.assert_array_equal(a, np.eye(6))
    assert not np.any(s)


def test_td_preserves_subdiagonal_storage():
    rng = np.random.default_rng(8)
    t0 = rng.standard_normal((6, 6))
    parked = np.tril(t0, -1).copy()
    t, _, _ = orc.comp_td_qr(t0, rng.standard_normal((6, 6)), 3)
    np.testing.assert_array_equal(np.tril(t, -1), parked)


# -- task lists (paper Tables II / III structure) --------------------------------------


def test_task_counts_closed_form_paper_grid():
    p, q = 27, 26  # the paper's 266,500 x 262,144 matrix at b = 10240
    tasks = orc.gen_factorization_tasks(p, q)
    assert len(tasks) == sum(k * p - k * (k - 1) // 2 + p - k for k in range(q))
    assert tasks[-1][0] == "comp_td_qr" and tasks[-1][1][:2] == (("A", 25, 25), ("A", 26, 25))


def test_task_lists_small_grids():
    assert [t[0] for t in orc.gen_factorization_tasks(2, 2)] == [
        "comp_dense_qr", "comp_td_qr", "apply_qt_dense", "apply_qt_td", "comp_dense_qr"]
    assert len(orc.gen_factorization_tasks(3, 3)) == 14
    ops = [t[0] for t in orc.gen_solve_tasks(2, 2, 1)]
    assert ops == ["apply_qt_dense", "apply_qt_td", "apply_qt_dense", "trsm_lunn",
                   "gemm_nn_mo", "trsm_lunn"]
    assert len(orc.gen_solve_tasks(3, 3, 1)) == 12


def test_dataflow_every_s_tile_written_before_read():
    rng = np.random.default_rng(7)
    for _ in range(10):
        p = int(rng.integers(1, 7))
        q = int(rng.integers(1, p + 1))
        produced = set()
        for _, outs, ins in orc.gen_factorization_tasks(p, q):
            assert all(ref in produced for ref in ins if ref[0] == "S")
            produced.update(outs)


# -- whole factorize / solve vs the reference run -------------------------------------


@pytest.mark.parametrize("idx", range(8))
def test_oracle_matches_reference_grid(golden, idx):
    g = golden("ref_grid.npz")
    m, n, b = (int(v) for v in g[f"g{idx}_shape"])
    f = orc.factorize_dense(g[f"g{idx}_a"], b, min(64, b))
    assert rel_err(sign_normalise(f.r()), g[f"g{idx}_r"]) <= 1e-12
    fw = orc.factorize_dense(g[f"g{idx}_aw"], b, min(64, b))
    x = orc.solve_dense(fw, g[f"g{idx}_b"])
    assert rel_err(x, g[f"g{idx}_x"]) <= 1e-12


@pytest.mark.parametrize("name", ["c6", "c3_19", "c0"])
def test_oracle_singular_column_order(golden, name):
    z = golden("ref_singular.npz")
    b = int(z[f"{name}_tile"][0])
    f = orc.factorize_dense(z[f"{name}_a"], b, min(64, b))
    with pytest.raises(orc.OracleSingularError) as e:
        orc.solve_dense(f, z[f"{name}_b"])
    assert e.value.global_column == int(z[f"{name}_col"][0])


@pytest.mark.parametrize("cfg", [0, 1])
def test_oracle_matches_reference_ct(golden, cfg):
    ref = golden(f"ref_ct{cfg}.npz")
    g = cs.config_geometry(cfg)
    a = cs.dense_matrix(g, order="C")
    # the generators must still produce the exact bytes the reference consumed
    import hashlib
    assert hashlib.sha256(a.tobytes()).hexdigest() == str(ref["a_sha256"])
    assert cs.geometry_hash(g) == str(ref["geometry_hash"])
    b, w = (int(v) for v in ref["tile"])
    f = orc.factorize_dense(a, b, w)
    x = orc.solve_dense(f, ref["b"])
    assert rel_err(x, ref["x"]) <= 1e-10
    np.testing.assert_allclose(np.abs(np.diag(f.r())), ref["rdiag_abs"], rtol=1e-12)
    resid = orc.residual_norms(f, ref["b"])
    np.testing.assert_allclose(resid, ref["resid"], rtol=1e-9)
    if "r_signed" in ref:
        assert rel_err(sign_normalise(f.r()), ref["r_signed"]) <= 1e-12
    else:
        assert rel_err(sign_normalise(f.r())[:32], ref["r_rows32"]) <= 1e-12


def test_config2_reference_fixture_inputs():
    """tests/golden/ref_ct2.npz (the reference package's factorize + solve of
    BASELINE config 2, make_golden_cfg2.py) was made from exactly the matrix
    and sinograms this repository generates: pinned by sha256."""
    import hashlib
    from pathlib import Path

    from paper_1907_01891_b200 import ct_system as cs
    ref = np.load(Path(__file__).resolve().parent / "golden" / "ref_ct2.npz")
    g = cs.config_geometry(2)
    assert str(ref["geometry_hash"]) == cs.geometry_hash(g)
    a = cs.dense_matrix(g, order="C")
    assert hashlib.sha256(a.tobytes()).hexdigest() == str(ref["a_sha256"])
    x_true = cs.phantom_stack(2, ref["b"].shape[1])
    b = cs.noisy_sinograms(a @ x_true, 2)
    assert np.array_equal(b, ref["b"])
    # the reference's residuals are those of its own solution
    assert np.allclose(np.linalg.norm(a @ ref["x"] - b, axis=0), ref["resid"], rtol=1e-12)


def test_quarter_width_config4_family_fixture_inputs():
    """tests/golden/ref_ct4q.npz (the reference package's factorize + solve of
    config 4's geometry family at 1/4 width, make_golden_cfg4q.py) was made
    from exactly the matrix and sinograms this repository generates."""
    import hashlib
    from pathlib import Path

    from paper_1907_01891_b200 import ct_system as cs
    ref = np.load(Path(__file__).resolve().parent / "golden" / "ref_ct4q.npz")
    g = cs.config_geometry(8)
    assert (g.n_rays, g.n_pixels) == (16920, 16384)
    assert str(ref["geometry_hash"]) == cs.geometry_hash(g)
    a = cs.dense_matrix(g, order="C")
    assert hashlib.sha256(a.tobytes()).hexdigest() == str(ref["a_sha256"])
    x_true = cs.phantom_stack(8, ref["b"].shape[1])
    b = cs.noisy_sinograms(a @ x_true, 8)
    assert np.array_equal(b, ref["b"])
    assert np.allclose(np.linalg.norm(a @ ref["x"] - b, axis=0), ref["resid"], rtol=1e-12)


def test_oracle_matches_reference_on_reduced_config4_family():
    """Config 4's geometry family at 1/8 width (ct_system CONFIGS[6], 4230 x 4096,
    m/n = 1.03 as at full size): the oracle's tiled factorization and solve
    equal the reference package's (tests/golden/make_golden_cfg4r.py) on the
    same bytes."""
    import hashlib
    from pathlib import Path

    from paper_1907_01891_b200 import ct_system as cs
    ref = np.load(Path(__file__).resolve().parent / "golden" / "ref_ct4r.npz")
    g = cs.config_geometry(6)
    assert str(ref["geometry_hash"]) == cs.geometry_hash(g)
    a = cs.dense_matrix(g, order="C")
    assert hashlib.sha256(a.tobytes()).hexdigest() == str(ref["a_sha256"])
    b = cs.noisy_sinograms(a @ cs.phantom_stack(6, ref["b"].shape[1]), 6)
    assert np.array_equal(b, ref["b"])
    f = orc.factorize_dense(a, 512, 128)
    x = orc.solve_dense(f, b)
    assert np.abs(x - ref["x"]).max() <= 1e-12 * np.abs(ref["x"]).max()
    r = f.r()
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    assert np.abs((r * s[:, None])[:8] - ref["r_rows8"]).max() <= 1e-12 * np.abs(ref["r_rows8"]).max()
