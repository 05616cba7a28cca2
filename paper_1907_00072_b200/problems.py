"""Problem inputs of the reference experiment runner (the
data formats on the caller's side of the path): the built-in test matrices,
their right-hand sides and the Matrix Market reader, restated so that
``cli.run_experiment`` assembles exactly the reference's problems
(sparse.py:151-440).  Host-side numpy; the solve itself runs on the device.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import MatrixFormatError, ParameterError
from .workloads import CsrHost, laplacian2d


class UnsupportedFormatError(MatrixFormatError):
    """The Matrix Market header requests an unsupported variant."""


class MatrixMarketParseError(MatrixFormatError):
    """Malformed Matrix Market data; ``line`` is 1-based."""

    def __init__(self, line, message):
        super().__init__(f"line {line}: {message}")
        self.line = line


def csr_from_coo(nrows, ncols, rows, cols, values) -> CsrHost:
    """Triplets -> CSR with rows sorted by (row, column) and duplicates summed
    in input order (CsrMatrix.from_coo, sparse.py:111-142)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    if not (rows.shape == cols.shape == values.shape):
        raise ParameterError("triplet arrays must have equal length")
    if len(rows) and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0
                      or cols.max() >= ncols):
        raise ParameterError("triplet indices out of range")
    order = np.lexsort((cols, rows))
    rows, cols, values = rows[order], cols[order], values[order]
    if len(rows):
        first = np.ones(len(rows), dtype=bool)
        first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        slot = np.cumsum(first) - 1
        acc = np.zeros(int(slot[-1]) + 1)
        np.add.at(acc, slot, values)
        rows, cols, values = rows[first], cols[first], acc
    counts = np.bincount(rows, minlength=nrows).astype(np.int64)
    row_ptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CsrHost(int(nrows), int(ncols), row_ptr, cols, values)


def gen_bidiag(n: int, diag_values, superdiag: float) -> CsrHost:
    """Upper bidiagonal: the given diagonal, constant superdiagonal
    (sparse.py:287-311); a zero superdiagonal stores the diagonal only."""
    if n < 1:
        raise ParameterError("empty matrix: n must be at least 1")
    d = np.asarray(diag_values, dtype=np.float64)
    if d.shape != (n,):
        raise ParameterError("diag_values must have length n")
    if superdiag == 0.0 or n == 1:
        return CsrHost(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
                       d.copy())
    per_row = np.full(n, 2, dtype=np.int64)
    per_row[-1] = 1
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(per_row, out=row_ptr[1:])
    cols = np.empty(2 * n - 1, dtype=np.int64)
    vals = np.empty(2 * n - 1)
    cols[0::2] = np.arange(n)
    cols[1::2] = np.arange(1, n)
    vals[0::2] = d
    vals[1::2] = superdiag
    return CsrHost(n, n, row_ptr, cols, vals)


def bidiag1() -> CsrHost:
    """n = 2000: diagonal 1..2000, superdiagonal 0.05 (sparse.py:314-316)."""
    return gen_bidiag(2000, np.arange(1, 2001, dtype=np.float64), 0.05)


def bidiag2() -> CsrHost:
    """n = 5000: diagonal 0.1..0.9, 1..4991, superdiagonal 0.2 (sparse.py:319-326)."""
    d = np.concatenate((np.arange(1, 10, dtype=np.float64) * 0.1,
                        np.arange(1, 4992, dtype=np.float64)))
    return gen_bidiag(5000, d, 0.2)


def gen_laplacian2d(grid_n: int) -> CsrHost:
    """Five-point Laplacian, 4 / -1, unscaled (sparse.py:329-359)."""
    return laplacian2d(grid_n)


def gen_laplacian_rhs(grid_n: int) -> np.ndarray:
    """Unit-source rhs: every entry h^2, h = 1/(g+1) (sparse.py:362-372)."""
    if grid_n < 1:
        raise ParameterError("empty matrix: grid_n must be at least 1")
    h = 1.0 / (grid_n + 1)
    return np.full(grid_n * grid_n, h * h)


def gen_convdiff2d(grid_n: int, epsilon: float):
    """Centred-difference ``-eps lap(u) + w.grad(u)`` on [-1, 1]^2 with the
    recirculating wind ``w = (2y(1-x^2), -2x(1-y^2))``, h^2-scaled, u = 1 on
    x = 1 folded into the rhs (sparse.py:375-433).  Returns (matrix, rhs)."""
    if epsilon <= 0.0:
        raise ParameterError("epsilon must be positive")
    if grid_n < 2:
        raise ParameterError("grid_n must be at least 2")
    g = grid_n
    n = g * g
    h = 2.0 / (g + 1)
    idx = np.arange(n, dtype=np.int64)
    i, j = idx % g, idx // g
    x = -1.0 + (i + 1) * h
    y = -1.0 + (j + 1) * h
    w1 = 2.0 * y * (1.0 - x * x)
    w2 = -2.0 * x * (1.0 - y * y)
    east = -epsilon + w1 * h / 2.0
    west = -epsilon - w1 * h / 2.0
    north = -epsilon + w2 * h / 2.0
    south = -epsilon - w2 * h / 2.0
    # row slots in increasing column order: south, west, centre, east, north
    slots = ((south, j > 0, -g), (west, i > 0, -1), (np.full(n, 4.0 * epsilon), None, 0),
             (east, i < g - 1, 1), (north, j < g - 1, g))
    mask = np.stack([np.ones(n, bool) if m is None else m for _, m, _ in slots], axis=1)
    vals = np.stack([c for c, _, _ in slots], axis=1)
    cols = idx[:, None] + np.array([o for _, _, o in slots], dtype=np.int64)[None, :]
    counts = mask.sum(axis=1, dtype=np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    matrix = CsrHost(n, n, row_ptr, cols[mask], vals[mask])
    rhs = np.zeros(n)
    wall = i == g - 1
    rhs[wall] = -east[wall]
    return matrix, rhs


def _lines(source):
    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            return fh.read().decode("latin-1").splitlines()
    if isinstance(source, bytes):
        return source.decode("latin-1").splitlines()
    data = source.read()
    return (data.decode("latin-1") if isinstance(data, bytes) else data).splitlines()


def read_matrix_market(source) -> CsrHost:
    """Matrix Market coordinate data (real / integer, general / symmetric)
    -> CSR, 0-based, rows sorted, duplicates summed (sparse.py:187-261)."""
    lines = _lines(source)
    if not lines:
        raise MatrixMarketParseError(1, "empty input")
    head = lines[0].split()
    if len(head) != 5 or not head[0].lower().startswith("%%matrixmarket"):
        raise MatrixMarketParseError(1, "malformed MatrixMarket banner")
    obj, fmt, field, sym = (t.lower() for t in head[1:])
    for what, got, ok in (("object", obj, ("matrix",)), ("format", fmt, ("coordinate",)),
                          ("field", field, ("real", "integer")),
                          ("symmetry", sym, ("general", "symmetric"))):
        if got not in ok:
            raise UnsupportedFormatError(f"unsupported {what} {got!r}")
    nr = nc = declared = -1
    rows, cols, vals = [], [], []
    seen = 0
    for ln, raw in enumerate(lines[1:], start=2):
        text = raw.strip()
        if not text or text.startswith("%"):
            continue
        tok = text.split()
        if declared < 0:
            if len(tok) != 3:
                raise MatrixMarketParseError(ln, "size line needs 3 integers")
            try:
                nr, nc, declared = (int(t) for t in tok)
            except ValueError:
                raise MatrixMarketParseError(ln, "size line needs 3 integers")
            if min(nr, nc, declared) < 0:
                raise MatrixMarketParseError(ln, "negative size entry")
            continue
        if seen >= declared:
            raise MatrixMarketParseError(ln, f"more than the declared {declared} entries")
        if len(tok) != 3:
            raise MatrixMarketParseError(ln, "entry needs 'row col value'")
        try:
            r, c, v = int(tok[0]), int(tok[1]), float(tok[2])
        except ValueError:
            raise MatrixMarketParseError(ln, f"cannot parse entry {text!r}")
        if not (1 <= r <= nr and 1 <= c <= nc):
            raise MatrixMarketParseError(ln, f"index ({r}, {c}) out of range")
        seen += 1
        rows.append(r - 1)
        cols.append(c - 1)
        vals.append(v)
        if sym == "symmetric" and r != c:
            rows.append(c - 1)
            cols.append(r - 1)
            vals.append(v)
    if declared < 0:
        raise MatrixMarketParseError(len(lines), "missing size line")
    if seen != declared:
        raise MatrixMarketParseError(len(lines), f"expected {declared} entries, found {seen}")
    return csr_from_coo(nr, nc, rows, cols, vals)
