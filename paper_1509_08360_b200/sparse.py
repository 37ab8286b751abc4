"""Host CSR container and input builders (host side of the boundary).

`SparseMatrix` keeps the reference's layout and invariants (sparse.py:55-99:
int64 row offsets / column indices, f64 values, sorted unique columns per row,
no stored zeros) so reference matrices and ours are interchangeable; the
device copy is made once per (matrix, dtype) and cached (see engine.py).

The builders (`normalized_adjacency`, `dilate`, `simple_edges`) reproduce the
reference's values bit-for-bit (same IEEE expressions, same canonical CSR
order) with sort-based numpy code that is O(T log T) instead of the
reference's 2-d `np.unique` pass.  They are host preprocessing, not part of
the measured recurrence.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def _frozen(a, dtype) -> np.ndarray:
    """A private read-only copy of `a` in `dtype` (the reference's immutable
    SparseMatrix arrays, sparse.py:20-25).  Large arrays are copied into
    pinned host memory, so the device upload (csemb_matrix_upload) is a
    direct DMA instead of a staged pageable copy."""
    src = np.asarray(a)
    if src.ndim == 1 and src.nbytes >= (1 << 20):
        out = _lib.host_empty(src.shape, dtype)
        np.copyto(out, src, casting="unsafe")
    else:
        out = np.ascontiguousarray(src, dtype=dtype)
        if out is src or out.base is src or np.shares_memory(out, src):
            out = out.copy()
    out.setflags(write=False)
    return out


class SparseMatrix:
    """Immutable CSR matrix (reference sparse.py:55-168 layout and checks)."""

    __slots__ = ("n_rows", "n_cols", "row_offsets", "col_indices", "values", "__weakref__")

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values, *, check: bool = True):
        if n_rows < 0 or n_cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        object.__setattr__(self, "n_rows", int(n_rows))
        object.__setattr__(self, "n_cols", int(n_cols))
        object.__setattr__(self, "row_offsets", _frozen(row_offsets, np.int64))
        object.__setattr__(self, "col_indices", _frozen(col_indices, np.int64))
        object.__setattr__(self, "values", _frozen(values, np.float64))
        if check:
            self._validate()

    def __setattr__(self, name, value):
        raise AttributeError("SparseMatrix is immutable")

    def _validate(self) -> None:
        offs, cols, vals = self.row_offsets, self.col_indices, self.values
        nnz = len(vals)
        if offs.shape != (self.n_rows + 1,):
            raise ValueError("row_offsets must have length n_rows + 1")
        if cols.shape != (nnz,):
            raise ValueError("col_indices and values must have equal length")
        if offs[0] != 0 or offs[-1] != nnz or (nnz and np.any(np.diff(offs) < 0)):
            raise ValueError("row_offsets must be non-decreasing from 0 to nnz")
        if nnz:
            if cols.min() < 0 or cols.max() >= self.n_cols:
                raise ValueError("column index out of range")
            starts = np.zeros(nnz, dtype=bool)
            inner = offs[1:-1]
            starts[inner[(inner > 0) & (inner < nnz)]] = True
            rising = cols[1:] > cols[:-1]
            if not np.all(rising | starts[1:]):
                raise ValueError("column indices must be strictly increasing per row")
            if np.any(vals == 0.0) or not np.all(np.isfinite(vals)):
                raise ValueError("stored values must be finite and nonzero")

    # -- construction ---------------------------------------------------------
    @classmethod
    def of(cls, S) -> "SparseMatrix":
        """Adopt any object with the reference's CSR attributes (no copy check)."""
        if isinstance(S, SparseMatrix):
            return S
        return cls(S.n_rows, S.n_cols, S.row_offsets, S.col_indices, S.values, check=False)

    @classmethod
    def from_scipy(cls, m) -> "SparseMatrix":
        import scipy.sparse as sp

        csr = sp.csr_array(m)
        csr.sum_duplicates()
        csr.sort_indices()
        csr.eliminate_zeros()
        return cls(csr.shape[0], csr.shape[1], csr.indptr.astype(np.int64),
                   csr.indices.astype(np.int64), csr.data.astype(np.float64))

    @classmethod
    def from_coo(cls, rows, cols, vals, n_rows: int, n_cols: int) -> "SparseMatrix":
        import scipy.sparse as sp

        coo = sp.coo_array((np.asarray(vals, dtype=np.float64),
                            (np.asarray(rows), np.asarray(cols))), shape=(n_rows, n_cols))
        return cls.from_scipy(coo)

    @classmethod
    def from_dense(cls, a, tol: float = 0.0) -> "SparseMatrix":
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("expected a 2-d array")
        r, c = np.nonzero(np.abs(a) > tol)
        return cls.from_coo(r, c, a[r, c], a.shape[0], a.shape[1])

    @classmethod
    def identity(cls, n: int) -> "SparseMatrix":
        i = np.arange(n, dtype=np.int64)
        return cls(n, n, np.arange(n + 1, dtype=np.int64), i, np.ones(n))

    @classmethod
    def zeros(cls, n_rows: int, n_cols: int) -> "SparseMatrix":
        return cls(n_rows, n_cols, np.zeros(n_rows + 1, dtype=np.int64),
                   np.empty(0, dtype=np.int64), np.empty(0))

    # -- views ----------------------------------------------------------------
    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def to_scipy(self):
        import scipy.sparse as sp

        return sp.csr_array((self.values, self.col_indices, self.row_offsets),
                            shape=(self.n_rows, self.n_cols))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out

    def __repr__(self):
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


def _csr_from_sorted_keys(keys: np.ndarray, vals: np.ndarray, n_rows: int, n_cols: int) -> SparseMatrix:
    """CSR from unique keys row*n_cols+col sorted ascending (canonical order)."""
    rows = keys // n_cols
    cols = keys - rows * n_cols
    offs = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=offs[1:])
    return SparseMatrix(n_rows, n_cols, offs, cols, vals, check=False)


def simple_edges(edges) -> np.ndarray:
    """Drop self-loops, collapse duplicates; rows (min, max) in lexicographic
    order (sparse.py:229-237)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    u, v = e[:, 0], e[:, 1]
    keep = u != v
    u, v = u[keep], v[keep]
    if len(u) == 0:
        return np.empty((0, 2), dtype=np.int64)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    n = int(hi.max()) + 1
    key = np.unique(lo * n + hi)
    return np.stack([key // n, key % n], axis=1)


def normalized_adjacency(edges, n: int) -> SparseMatrix:
    """D^{-1/2} A D^{-1/2} of the simple graph (sparse.py:202-226): entry
    1/sqrt(deg u * deg v), isolated vertices keep zero rows."""
    if n < 1:
        raise ValueError("vertex count must be positive")
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ValueError("edge endpoint out of range [0, n)")
    u, v = e[:, 0], e[:, 1]
    keep = u != v
    u, v = u[keep], v[keep]
    if len(u) == 0:
        return SparseMatrix.zeros(n, n)
    key = np.unique(np.minimum(u, v) * n + np.maximum(u, v))
    lo, hi = key // n, key % n
    deg = np.bincount(lo, minlength=n) + np.bincount(hi, minlength=n)
    degf = deg.astype(np.float64)
    # both orientations, canonical (row, col) order
    sym = np.concatenate([lo * n + hi, hi * n + lo])
    order = np.argsort(sym, kind="stable")
    sym = sym[order]
    r, c = sym // n, sym % n
    vals = 1.0 / np.sqrt(degf[r] * degf[c])
    return _csr_from_sorted_keys(sym, vals, n, n)


def dilate(A) -> SparseMatrix:
    """[0 A^T; A 0]: the first n indices are A's columns, the last m its rows
    (sparse.py:191-199)."""
    A = SparseMatrix.of(A)
    if A.n_rows < 1 or A.n_cols < 1:
        raise ValueError("cannot dilate an empty matrix")
    m, n = A.n_rows, A.n_cols
    N = m + n
    r = np.repeat(np.arange(m, dtype=np.int64), np.diff(A.row_offsets))
    c = A.col_indices
    # A^T block: rows c, cols n + r ; A block: rows n + r, cols c
    keys = np.concatenate([c * N + (n + r), (n + r) * N + c])
    vals = np.concatenate([A.values, A.values])
    order = np.argsort(keys, kind="stable")
    return _csr_from_sorted_keys(keys[order], vals[order], N, N)


def scale_values(S, factor: float) -> SparseMatrix:
    """S * factor on the values (sparse.py:295-301)."""
    if factor == 0.0 or not np.isfinite(factor):
        raise ValueError("scale factor must be finite and nonzero")
    S = SparseMatrix.of(S)
    return SparseMatrix(S.n_rows, S.n_cols, S.row_offsets, S.col_indices, S.values * factor,
                        check=False)
