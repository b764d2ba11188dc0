"""Host-side drop-in logic and the C-ABI boundary, without launching GPU work."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1907_01891_b200 as pkg
from paper_1907_01891_b200 import _native, build
from paper_1907_01891_b200.task_engine import EngineConfig, factorize

HEADER = Path(__file__).resolve().parent.parent / "include" / "qrb200.h"


def header_symbols():
    return set(re.findall(r"QRB_API\s+[\w\s\*]+?\b(qrb_\w+)\s*\(", HEADER.read_text()))


def test_reference_public_names_exported():
    for name in ["TileCache", "TiledMatrix", "TileId", "EngineConfig", "RunReport",
                 "factorize", "solve"]:
        assert hasattr(pkg, name), name
    assert issubclass(pkg.KernelInputError, ValueError)
    assert pkg.SingularMatrixError(6).global_column == 6
    assert pkg.TaskIoError(3, "op", OSError("x")).seq == 3


def test_ctypes_table_matches_header():
    syms = header_symbols()
    assert len(syms) >= 18
    assert syms == set(_native.SIGNATURES)


def test_library_builds_loads_and_exports_every_symbol():
    lib_path = build.build()
    assert lib_path.exists()
    lib = _native.load()
    for sym in header_symbols():
        assert hasattr(lib, sym), sym
    assert lib.qrb_version() >= 100


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_LIB_PATH", tmp_path / "libqrb200.so")
    monkeypatch.setattr(_native, "_lib", None)
    from paper_1907_01891_b200.device import QrDevice
    with pytest.raises(pkg.NativeUnavailableError):
        QrDevice(8, 8)


def test_engine_config_validation():
    for bad in [dict(tile_size=0), dict(tile_size=8, inner_block=9), dict(mode="parallel"),
                dict(mode="overlapped", io_agents=2), dict(compute_workers=0),
                dict(prefetch_depth=-1), dict(panel_width=100), dict(panel_width=256)]:
        with pytest.raises(ValueError):
            EngineConfig(**bad).validate()
    assert EngineConfig().validate() is not None
    assert EngineConfig(mode="overlapped", prefetch_depth=2).min_cache_tiles() == 14


def test_factorize_argument_errors_before_device(tmp_path):
    a = pkg.TiledMatrix.create(4, 8, 4, tmp_path / "a")
    with pytest.raises(ValueError, match="rows >= cols"):
        factorize(a, EngineConfig(tile_size=4, inner_block=4), tmp_path / "f")
    a = pkg.TiledMatrix.create(8, 8, 4, tmp_path / "a2")
    with pytest.raises(ValueError, match="tile_size"):
        factorize(a, EngineConfig(tile_size=8, inner_block=4), tmp_path / "f")


def test_factors_meta_marks_algorithm(tmp_path):
    from paper_1907_01891_b200.task_engine import QrFactors
    m = pkg.TiledMatrix.create(8, 8, 4, tmp_path / "f" / "factored")
    f = QrFactors(factored=m, inner_block=4, rows=8, cols=8, tile_size=4, panel_width=128,
                  geometry_hash="abc", directory=tmp_path / "f")
    f.save_meta(tmp_path / "f")
    text = (tmp_path / "f" / "meta.txt").read_text()
    assert "algorithm geqrf_cwy" in text and "geometry_hash abc" in text
    g = QrFactors.load(tmp_path / "f")
    assert (g.rows, g.cols, g.tile_size, g.inner_block, g.geometry_hash) == (8, 8, 4, 4, "abc")
    with pytest.raises(pkg.MissingFactorsError):
        g.check_complete()
    with pytest.raises(pkg.MissingFactorsError):
        QrFactors.load(tmp_path / "nope")
    # a reference-format meta (no algorithm key) is refused, never misread
    (tmp_path / "r").mkdir()
    (tmp_path / "r" / "meta.txt").write_text("rows 8\ncols 8\ntile_size 4\ninner_block 4\n"
                                             "geometry_hash -\n")
    with pytest.raises(pkg.MissingFactorsError):
        QrFactors.load(tmp_path / "r")


def test_singular_rule_matches_reference_order():
    # the C library applies the rule; its host-side twin is exercised on GPU.
    # Here: the reference rule on a synthetic diagonal, restated for clarity.
    diag = np.ones(24)
    diag[[3, 19]] = 0.0
    block = 8
    bad_tiles = sorted({i // block for i in np.flatnonzero(np.abs(diag) < 1e-300)})
    t = bad_tiles[-1]
    first = next(i for i in range(t * block, (t + 1) * block) if abs(diag[i]) < 1e-300)
    assert first == 19


def test_column_reader_flags_chunks_in_order_and_aborts_on_a_bad_tile(tmp_path):
    """The drop-in factorize's tile reader (task_engine._ColumnReader) raises a
    chunk's ready flag only once every column of the chunk is in the host
    matrix, and marks every pending chunk -1 (so the native call returns
    instead of waiting) when a tile cannot be read."""
    import numpy as np
    import paper_1907_01891_b200 as pkg
    from paper_1907_01891_b200.task_engine import _ColumnReader
    rng = np.random.default_rng(2)
    m, n, b = 50, 70, 16
    a = rng.standard_normal((m, n))
    t = pkg.TiledMatrix.create(m, n, b, tmp_path / "a")
    pkg.scatter_matrix(t, a)
    lda = 64
    host = np.zeros((n, lda))
    ready = np.zeros(-(-n // 24), dtype=np.int32)          # chunks of 24 columns
    r = _ColumnReader(t, host.T, 24, ready, threads=3)
    r.start()
    r.join()
    assert (ready == 1).all()
    np.testing.assert_array_equal(host.T[:m], a)
    # a truncated tile: TaskIoError, and no chunk is left waiting
    t.tile_path(pkg.TileId(1, 2)).write_bytes(b"\0" * 8)
    ready[:] = 0
    r = _ColumnReader(t, np.zeros((n, lda)).T, 24, ready, threads=2)
    r.start()
    with pytest.raises(pkg.TaskIoError):
        r.join()
    assert (ready != 0).all() and (ready == -1).any()
