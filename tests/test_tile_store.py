"""Drop-in tile store: the reference's on-disk format (tile_store.py:25-30, 132-209)."""

import struct

import numpy as np
import pytest

from paper_1907_01891_b200 import (CacheCapacityError, CorruptTileError, ManifestError,
                                   TileCache, TiledMatrix, TileId, gather_matrix,
                                   scatter_matrix)


def test_manifest_keys_in_reference_order(tmp_path):
    TiledMatrix.create(13, 7, 5, tmp_path / "m")
    lines = (tmp_path / "m" / "manifest.txt").read_text().splitlines()
    assert lines == ["format_version 1", "element_type f64le", "order col-major",
                     "rows 13", "cols 7", "tile_size 5"]
    m = TiledMatrix.open(tmp_path / "m")
    assert (m.rows, m.cols, m.tile_size, m.grid_rows, m.grid_cols) == (13, 7, 5, 3, 2)


def test_paper_grid_without_tiles(tmp_path):
    m = TiledMatrix.create(266_500, 262_144, 10_240, tmp_path / "big")
    assert (m.grid_rows, m.grid_cols) == (27, 26)
    assert not list(m.directory.glob("*.blk"))


def test_tile_bytes_column_major_little_endian(tmp_path):
    m = TiledMatrix.create(2, 2, 2, tmp_path / "m")
    m.store_tile(TileId(0, 0), np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert m.tile_path(TileId(0, 0)).read_bytes() == struct.pack("<4d", 1.0, 3.0, 2.0, 4.0)


def test_round_trip_padding_absent_corrupt(tmp_path):
    rng = np.random.default_rng(7)
    m = TiledMatrix.create(10, 10, 4, tmp_path / "m")
    m.store_tile(TileId(2, 2), np.full((4, 4), 5.0))
    back = m.load_tile(TileId(2, 2))
    assert np.all(back[:2, :2] == 5.0) and not back[2:, :].any() and not back[:, 2:].any()
    assert not m.load_tile(TileId(1, 1)).any()
    buf = rng.standard_normal((4, 4))
    m.store_tile(TileId(0, 0), buf)
    assert m.load_tile(TileId(0, 0)).tobytes() == buf.tobytes()
    p = m.tile_path(TileId(0, 0))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(CorruptTileError):
        m.load_tile(TileId(0, 0))
    with pytest.raises(CorruptTileError):
        m.read_column_block(0)
    with pytest.raises(IndexError):
        m.load_tile(TileId(3, 0))


def test_manifest_errors(tmp_path):
    with pytest.raises(ManifestError):
        TiledMatrix.open(tmp_path / "nope")
    TiledMatrix.create(8, 8, 4, tmp_path / "m")
    with pytest.raises(ManifestError):
        TiledMatrix.create(8, 8, 2, tmp_path / "m")
    (tmp_path / "bad").mkdir()
    (tmp_path / "bad" / "manifest.txt").write_text("rows ten\ncols 4\n")
    with pytest.raises(ManifestError):
        TiledMatrix.open(tmp_path / "bad")


@pytest.mark.parametrize("shape,b", [((13, 9), 4), ((8, 8), 8), ((5, 3), 8), ((33, 20), 7)])
def test_scatter_gather_and_column_blocks(tmp_path, shape, b):
    rng = np.random.default_rng(shape[0])
    a = rng.standard_normal(shape)
    m = TiledMatrix.create(*shape, b, tmp_path / "m")
    scatter_matrix(m, a)
    np.testing.assert_array_equal(gather_matrix(m), a)
    for j in range(m.grid_cols):
        np.testing.assert_array_equal(m.read_column_block(j), a[:, j * b:(j + 1) * b])
    # via the cache as well
    cache = TileCache(64)
    np.testing.assert_array_equal(gather_matrix(m, cache), a)


def test_cache_lru_pins_and_flush(tmp_path):
    m = TiledMatrix.create(12, 4, 4, tmp_path / "m")
    for i in range(3):
        m.store_tile(TileId(i, 0), np.full((4, 4), float(i + 1)))
    c = TileCache(2)
    c.acquire(m, TileId(0, 0))
    c.acquire(m, TileId(1, 0))
    c.acquire(m, TileId(2, 0))  # evicts (0,0)
    assert not c.is_resident(m, TileId(0, 0))
    assert c.reads_from_disk == 3 and c.hits == 0
    c.acquire(m, TileId(1, 0), pin=True)
    c.acquire(m, TileId(2, 0), pin=True)
    with pytest.raises(CacheCapacityError):
        c.acquire(m, TileId(0, 0))
    c.release(m, TileId(1, 0))
    c.release(m, TileId(2, 0))
    c.put(m, TileId(0, 0), np.zeros((4, 4)))
    c.flush()
    assert not m.load_tile(TileId(0, 0)).any()
    assert c.writes_to_disk == 1


def test_uncached_column_io_roundtrip(tmp_path):
    """Page-cache-bypassing column I/O (the disk tier's uncached mode) moves the
    same bytes as the cached path."""
    from paper_1907_01891_b200.tile_store import TiledMatrix
    rng = np.random.default_rng(4)
    m, n, b = 70, 45, 16
    a = rng.standard_normal((m, n))
    t = TiledMatrix.create(m, n, b, tmp_path / "u")
    t.uncached = True
    t.write_columns(0, n, np.asfortranarray(a))
    out = np.zeros((m, 20), order="F")
    t.read_columns(13, 20, 5, out)
    np.testing.assert_array_equal(out[5:], a[5:, 13:33])
    assert not out[:5].any()
