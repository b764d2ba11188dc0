"""Numpy restatement of the reference tiled QR / solve (oracle; tests only).

Follows pkg/src/oocqr/kernels.py and task_engine.py of the reference:

* Householder convention (dlarfg-like, no rescaling)       kernels.py:74-77
* dense-tile panel + T builder                              kernels.py:80-101, 134-147
* triangle-on-dense (TD) panel + T builder                  kernels.py:172-193, 226-235
* comp_dense_qr / apply_left_qt_dense                       kernels.py:296-341
* comp_td_qr / apply_left_qt_td                             kernels.py:344-405
* trsm_lunn (singular floor 1e-300, padded rows zeroed)     kernels.py:408-439
* gemm_nn_mo                                                kernels.py:442-455
* left-looking task lists (paper Tables II / III)           task_engine.py:187-254
* task dispatch incl. TRSM extent / col_offset              task_engine.py:287-317

The tile store is kept in memory (a dict of b x b arrays) instead of on disk;
the arithmetic and its order per tile are the reference's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SINGULAR_FLOOR = 1e-300  # kernels.py:36


class OracleInputError(ValueError):
    """Shape / finiteness violation (reference KernelInputError, kernels.py:40-41)."""


class OracleSingularError(RuntimeError):
    """Reference SingularMatrixError (kernels.py:44-52)."""

    def __init__(self, global_column: int):
        self.global_column = int(global_column)
        super().__init__(f"zero pivot at global column {self.global_column}")


# -- Householder machinery ----------------------------------------------------


def _reflector(alpha: float, sigma: float):
    """(beta, tau, 1/(alpha-beta)) for x = [alpha; x2], sigma = |x2|^2; None if sigma == 0."""
    if sigma == 0.0:
        return None
    beta = -math.copysign(math.sqrt(alpha * alpha + sigma), alpha)
    return beta, (beta - alpha) / beta, 1.0 / (alpha - beta)


def _factor_columns(rows_of, j0: int, pw: int) -> np.ndarray:
    """Column-by-column Householder sweep over panel columns [j0, j0+pw).

    ``rows_of(col)`` returns (pivot row 1-D view, 2-D view of the rows the
    reflector reaches below it).  Dense tiles: (a[col], a[col+1:]); TD pairs:
    (t[col], d).
    """
    taus = np.zeros(pw)
    end = j0 + pw
    for k in range(pw):
        col = j0 + k
        head, tail = rows_of(col)
        x = tail[:, col]
        h = _reflector(head[col], float(x @ x))
        if h is None:
            continue
        beta, tau, scale = h
        x *= scale
        head[col] = beta
        taus[k] = tau
        if col + 1 < end:
            right = slice(col + 1, end)
            srow = (head[right] + x @ tail[:, right]) * tau
            head[right] -= srow
            tail[:, right] -= np.outer(x, srow)
    return taus


def _t_factor(gram, taus: np.ndarray) -> np.ndarray:
    """Upper-triangular T with T[k,k] = tau_k, T[:k,k] = -tau_k T[:k,:k] gram(k)."""
    pw = taus.size
    t = np.zeros((pw, pw))
    for k in range(pw):
        t[k, k] = taus[k]
        if k > 0 and taus[k] != 0.0:
            t[:k, k] = -taus[k] * (t[:k, :k] @ gram(k))
    return t


def _unit_lower(a: np.ndarray, j0: int, pw: int) -> np.ndarray:
    v = np.tril(a[j0:, j0:j0 + pw], -1)
    v[np.arange(pw), np.arange(pw)] = 1.0
    return v


def _check_square(name, t, b=None):
    if t.ndim != 2 or t.shape[0] != t.shape[1] or (b is not None and t.shape[0] != b):
        raise OracleInputError(f"{name} must be a square tile, got {t.shape}")
    return t.shape[0]


def _check_w(w, b):
    if not 1 <= int(w) <= b:
        raise OracleInputError(f"inner block width must be in [1, {b}], got {w}")
    return int(w)


# -- the six tile kernels ----------------------------------------------------------


def comp_dense_qr(a: np.ndarray, w: int):
    """In-place Householder QR of one tile; returns (a, s) with s the packed T tile."""
    b = _check_square("a", a)
    w = _check_w(w, b)
    if not np.isfinite(a).all():
        raise OracleInputError("comp_dense_qr: non-finite tile")
    s = np.zeros((b, b))
    for j0 in range(0, b, w):
        pw = min(w, b - j0)
        taus = _factor_columns(lambda c: (a[c], a[c + 1:]), j0, pw)

        def gram(k, j0=j0):
            col = j0 + k
            return a[col, j0:col] + a[col + 1:, j0:col].T @ a[col + 1:, col]

        t = _t_factor(gram, taus)
        s[j0:j0 + pw, :pw] = t
        if j0 + pw < b:
            v = _unit_lower(a, j0, pw)
            a[j0:, j0 + pw:] -= v @ (t.T @ (v.T @ a[j0:, j0 + pw:]))
    return a, s


def apply_left_qt_dense(y: np.ndarray, s: np.ndarray, c: np.ndarray, w: int) -> np.ndarray:
    b = _check_square("y", y)
    _check_square("s", s, b)
    w = _check_w(w, b)
    if c.ndim != 2 or c.shape[0] != b:
        raise OracleInputError(f"c must have {b} rows")
    for j0 in range(0, b, w):
        pw = min(w, b - j0)
        v = _unit_lower(y, j0, pw)
        t = s[j0:j0 + pw, :pw]
        c[j0:, :] -= v @ (t.T @ (v.T @ c[j0:, :]))
    return c


def comp_td_qr(t: np.ndarray, d: np.ndarray, w: int):
    """QR of [upper(t); d] in place; returns (t, d, s)."""
    b = _check_square("t", t)
    _check_square("d", d, b)
    w = _check_w(w, b)
    if not np.isfinite(d).all():
        raise OracleInputError("comp_td_qr: non-finite tile")
    s = np.zeros((b, b))
    for j0 in range(0, b, w):
        pw = min(w, b - j0)
        taus = _factor_columns(lambda c: (t[c], d), j0, pw)
        tf = _t_factor(lambda k, j0=j0: d[:, j0:j0 + k].T @ d[:, j0 + k], taus)
        s[j0:j0 + pw, :pw] = tf
        end = j0 + pw
        if end < b:
            vd = d[:, j0:end]
            z = tf.T @ (t[j0:end, end:] + vd.T @ d[:, end:])
            t[j0:end, end:] -= z
            d[:, end:] -= vd @ z
    return t, d, s


def apply_left_qt_td(d: np.ndarray, s: np.ndarray, f: np.ndarray, g: np.ndarray, w: int):
    b = _check_square("d", d)
    _check_square("s", s, b)
    w = _check_w(w, b)
    for j0 in range(0, b, w):
        pw = min(w, b - j0)
        vd = d[:, j0:j0 + pw]
        z = s[j0:j0 + pw, :pw].T @ (f[j0:j0 + pw, :] + vd.T @ g)
        f[j0:j0 + pw, :] -= z
        g -= vd @ z
    return f, g


def trsm_lunn(rt: np.ndarray, bmat: np.ndarray, extent: int | None = None,
              col_offset: int = 0, block: int = 128) -> np.ndarray:
    """bmat <- upper(rt)^-1 bmat on the leading `extent` rows, rest zeroed."""
    b = _check_square("rt", rt)
    n = b if extent is None else int(extent)
    diag = np.abs(np.diagonal(rt)[:n])
    bad = np.flatnonzero(~(diag >= SINGULAR_FLOOR))
    if bad.size:
        raise OracleSingularError(col_offset + int(bad[0]))
    hi = n
    while hi > 0:
        lo = max(0, hi - block)
        for i in range(hi - 1, lo - 1, -1):
            if i + 1 < hi:
                bmat[i, :] -= rt[i, i + 1:hi] @ bmat[i + 1:hi, :]
            bmat[i, :] /= rt[i, i]
        if lo > 0:
            bmat[:lo, :] -= rt[:lo, lo:hi] @ bmat[lo:hi, :]
        hi = lo
    bmat[n:, :] = 0.0
    return bmat


def gemm_nn_mo(c: np.ndarray, a: np.ndarray, bmat: np.ndarray) -> np.ndarray:
    c -= a @ bmat
    return c


# -- task lists (paper Tables II / III) --------------------------------------------------


def gen_factorization_tasks(p: int, q: int):
    """Left-looking tiled QR: list of (op, outs, ins) (task_engine.py:187-217)."""
    if not p >= q >= 1:
        raise ValueError("grid must satisfy rows >= cols >= 1")
    out = []
    for k in range(q):
        for j in range(k):
            out.append(("apply_qt_dense", (("A", j, k),), (("A", j, j), ("S", j, j), ("A", j, k))))
            for i in range(j + 1, p):
                out.append(("apply_qt_td", (("A", j, k), ("A", i, k)),
                            (("A", i, j), ("S", i, j), ("A", j, k), ("A", i, k))))
        out.append(("comp_dense_qr", (("A", k, k), ("S", k, k)), (("A", k, k),)))
        for i in range(k + 1, p):
            out.append(("comp_td_qr", (("A", k, k), ("A", i, k), ("S", i, k)),
                        (("A", k, k), ("A", i, k))))
    return out


def gen_solve_tasks(p: int, q: int, r: int):
    """Per RHS block column: Q^T applies, then bottom-up back substitution
    (task_engine.py:220-254)."""
    if not p >= q >= 1 or r < 1:
        raise ValueError("bad grid")
    out = []
    for c in range(r):
        for k in range(q):
            out.append(("apply_qt_dense", (("B", k, c),), (("A", k, k), ("S", k, k), ("B", k, c))))
            for i in range(k + 1, p):
                out.append(("apply_qt_td", (("B", k, c), ("B", i, c)),
                            (("A", i, k), ("S", i, k), ("B", k, c), ("B", i, c))))
        for k in range(q - 1, -1, -1):
            for j in range(k + 1, q):
                out.append(("gemm_nn_mo", (("B", k, c),), (("B", k, c), ("A", k, j), ("B", j, c))))
            out.append(("trsm_lunn", (("B", k, c),), (("A", k, k), ("B", k, c))))
    return out


# -- in-memory executor ------------------------------------------------------------------


def _to_tiles(arr: np.ndarray, b: int) -> dict:
    m, n = arr.shape
    tiles = {}
    for i in range(-(-m // b)):
        for j in range(-(-n // b)):
            t = np.zeros((b, b))
            blk = arr[i * b:(i + 1) * b, j * b:(j + 1) * b]
            t[:blk.shape[0], :blk.shape[1]] = blk
            tiles[(i, j)] = t
    return tiles


def _from_tiles(tiles: dict, m: int, n: int, b: int) -> np.ndarray:
    out = np.zeros((m, n))
    for (i, j), t in tiles.items():
        r, c = min(b, m - i * b), min(b, n - j * b)
        if r > 0 and c > 0:
            out[i * b:i * b + r, j * b:j * b + c] = t[:r, :c]
    return out


def _run(tasks, stores: dict, w: int, cols: int, b: int) -> None:
    for op, outs, ins in tasks:
        if op == "comp_dense_qr":
            (ra,) = ins
            _, s = comp_dense_qr(stores[ra[0]][ra[1:]], w)
            stores["S"][outs[1][1:]] = s
        elif op == "comp_td_qr":
            rt, rd = ins
            _, _, s = comp_td_qr(stores["A"][rt[1:]], stores["A"][rd[1:]], w)
            stores["S"][outs[2][1:]] = s
        elif op == "apply_qt_dense":
            ry, rs, rc = ins
            apply_left_qt_dense(stores["A"][ry[1:]], stores["S"][rs[1:]],
                                stores[rc[0]][rc[1:]], w)
        elif op == "apply_qt_td":
            rd, rs, rf, rg = ins
            apply_left_qt_td(stores["A"][rd[1:]], stores["S"][rs[1:]],
                             stores[rf[0]][rf[1:]], stores[rg[0]][rg[1:]], w)
        elif op == "trsm_lunn":
            ra, rb = ins
            k = ra[2]
            extent = min(b, cols - k * b)
            trsm_lunn(stores["A"][ra[1:]], stores["B"][rb[1:]], extent=extent,
                      col_offset=k * b, block=w)
        elif op == "gemm_nn_mo":
            rc, ra, rb = ins
            gemm_nn_mo(stores["B"][rc[1:]], stores["A"][ra[1:]], stores["B"][rb[1:]])
        else:  # pragma: no cover
            raise ValueError(op)


@dataclass
class OracleFactors:
    rows: int
    cols: int
    tile_size: int
    inner_block: int
    a_tiles: dict = field(repr=False)
    s_tiles: dict = field(repr=False)

    def factored(self) -> np.ndarray:
        return _from_tiles(self.a_tiles, self.rows, self.cols, self.tile_size)

    def r(self) -> np.ndarray:
        return np.triu(self.factored()[: self.cols, :])


def factorize_dense(a: np.ndarray, tile_size: int, inner_block: int) -> OracleFactors:
    """Reference factorize() on an in-memory copy of a dense matrix."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m < n:
        raise ValueError("rows >= cols required")
    b = int(tile_size)
    tiles = _to_tiles(a, b)
    p, q = -(-m // b), -(-n // b)
    stores = {"A": tiles, "S": {}}
    _run(gen_factorization_tasks(p, q), stores, int(inner_block), n, b)
    return OracleFactors(m, n, b, int(inner_block), stores["A"], stores["S"])


def solve_dense(f: OracleFactors, bmat: np.ndarray) -> np.ndarray:
    """Reference solve(): X = R^-1 (Q^T B)[:n]; B padded to whole tile columns."""
    bmat = np.asarray(bmat, dtype=np.float64)
    if bmat.ndim == 1:
        bmat = bmat[:, None]
    b = f.tile_size
    p, q = -(-f.rows // b), -(-f.cols // b)
    r = -(-bmat.shape[1] // b)
    btiles = _to_tiles(bmat, b)
    for i in range(p):
        for c in range(r):
            btiles.setdefault((i, c), np.zeros((b, b)))
    stores = {"A": f.a_tiles, "S": f.s_tiles, "B": btiles}
    _run(gen_solve_tasks(p, q, r), stores, f.inner_block, f.cols, b)
    x_tiles = {(k, c): btiles[(k, c)] for k in range(q) for c in range(r)}
    return _from_tiles(x_tiles, f.cols, bmat.shape[1], b)


def residual_norms(f: OracleFactors, bmat: np.ndarray) -> np.ndarray:
    """||(Q^T B)[n:m, j]|| via the Q^T-only part of the solve task list."""
    bmat = np.asarray(bmat, dtype=np.float64)
    if bmat.ndim == 1:
        bmat = bmat[:, None]
    b = f.tile_size
    p, q = -(-f.rows // b), -(-f.cols // b)
    r = -(-bmat.shape[1] // b)
    btiles = _to_tiles(bmat, b)
    for i in range(p):
        for c in range(r):
            btiles.setdefault((i, c), np.zeros((b, b)))
    qt_only = [t for t in gen_solve_tasks(p, q, r) if t[0].startswith("apply")]
    stores = {"A": f.a_tiles, "S": f.s_tiles, "B": btiles}
    _run(qt_only, stores, f.inner_block, f.cols, b)
    qtb = _from_tiles(btiles, f.rows, bmat.shape[1], b)
    return np.linalg.norm(qtb[f.cols:, :], axis=0)
