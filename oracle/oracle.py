"""ctypes front end of the C oracle plus small numpy restatements.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Each function names the
reference file:line it restates (reference = /root/reference/pkg/src/csemb).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

NORM_SEED_TAG = 0x6E6F726D  # engine.py:36


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "csemb_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-B", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            L.oracle_mix64.restype = C.c_uint64
            L.oracle_mix64.argtypes = [C.c_uint64]
            L.oracle_fold_seed.restype = C.c_uint64
            L.oracle_fold_seed.argtypes = [C.c_uint64, C.c_uint64]
            L.oracle_sample_projection.restype = C.c_int
            L.oracle_sample_projection.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, _f64p]
            L.oracle_spmm.restype = C.c_int
            L.oracle_spmm.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int64, _f64p]
            L.oracle_run_stage.restype = C.c_int
            L.oracle_run_stage.argtypes = [
                C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int, _f64p, C.c_int64, _f64p,
                C.c_void_p, C.POINTER(C.c_int),
            ]
            L.oracle_num_threads.restype = C.c_int
            L.oracle_set_threads.argtypes = [C.c_int]
            _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


class CSR:
    """Plain CSR triple (int64 offsets/indices, f64 values) for the oracle."""

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)

    @classmethod
    def of(cls, S):
        if isinstance(S, CSR):
            return S
        return cls(S.n_rows, S.n_cols, S.row_offsets, S.col_indices, S.values)

    @property
    def nnz(self):
        return len(self.values)


# -- projection block ---------------------------------------------------------

def fold_seed(seed: int, index: int) -> int:
    """engine.fold_seed (engine.py:53-56)."""
    M = (1 << 64) - 1
    return int(lib().oracle_fold_seed(seed & M, index & M))


def sample_projection(n: int, d: int, seed: int, col0: int = 0, w: int | None = None) -> np.ndarray:
    """engine.sample_projection (engine.py:79-99), optionally a column slice
    [col0, col0+w) hashed with the GLOBAL d (engine.py:96)."""
    w = d - col0 if w is None else w
    out = np.empty((n, w), dtype=np.float64)
    rc = lib().oracle_sample_projection(n, d, seed & ((1 << 64) - 1), col0, w, out)
    if rc:
        raise ValueError("bad projection shape")
    return out


def np_sample_projection(n: int, d: int, seed: int) -> np.ndarray:
    """Pure-numpy restatement of the same hash (cross-check of the C port)."""
    def mix(z):
        with np.errstate(over="ignore"):
            z = z + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))
    key = mix(np.uint64(seed & ((1 << 64) - 1)))
    idx = np.arange(n, dtype=np.uint64)[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)
    h = mix(idx ^ key)
    s = 1.0 / math.sqrt(d)
    return np.where((h >> np.uint64(63)) & np.uint64(1), s, -s)


# -- SpMM and the recurrence ----------------------------------------------------

def spmm(S, X: np.ndarray) -> np.ndarray:
    """sparse.spmv_multi (sparse.py:171-188) == scipy csr_matvecs order."""
    S = CSR.of(S)
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim == 1:
        return spmm(S, X[:, None])[:, 0]
    if X.shape[0] != S.n_cols:
        raise ValueError("dimension mismatch")
    Y = np.empty((S.n_rows, X.shape[1]), dtype=np.float64)
    lib().oracle_spmm(S.n_rows, S.row_offsets, S.col_indices, S.values, X, X.shape[1], Y)
    return Y


def run_stage(S, coeffs, block):
    """engine._run_stage over the whole block (engine.py:205-228).

    Returns (out, max_abs[order, n_chunks], first_bad_r); column chunking
    (engine.py:242) does not change values, only the per-chunk peaks.
    """
    S = CSR.of(S)
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    block = np.ascontiguousarray(block, dtype=np.float64)
    n, w = block.shape
    order = len(coeffs) - 1
    out = np.empty_like(block)
    n_chunks = (w + 31) // 32
    peaks = np.zeros((max(order, 1), max(n_chunks, 1)), dtype=np.float64)
    bad = C.c_int(0)
    rc = lib().oracle_run_stage(
        n, S.row_offsets, S.col_indices, S.values, coeffs, order, block, w, out,
        peaks.ctypes.data_as(C.c_void_p), C.byref(bad),
    )
    if rc:
        raise MemoryError("oracle allocation failed")
    return out, peaks[:order, :n_chunks], int(bad.value)


def apply_expansion(S, coeffs, block, n_stages: int = 1):
    """engine._apply_expansion chained over cascade stages (engine.py:231-258,
    332-336).  Returns (out, first_bad_r of the first failing stage, stage)."""
    out = np.ascontiguousarray(block, dtype=np.float64)
    for st in range(1, n_stages + 1):
        out, _, bad = run_stage(S, coeffs, out)
        if bad:
            return out, bad, st
    return out, 0, 0


# -- norm estimate, normalisation, pair sampling --------------------------------

def spectral_norm(S, seed: int, iters: int = 20, factor: float = 6.0, safety: float = 1.01,
                  v0: np.ndarray | None = None) -> float:
    """engine.estimate_spectral_norm (engine.py:165-192), SpMM via the oracle."""
    S = CSR.of(S)
    if S.nnz == 0:
        return 0.0
    n = S.n_rows
    k = max(1, math.ceil(factor * math.log(max(n, 2))))
    if v0 is None:
        V = np.random.default_rng(fold_seed(seed, NORM_SEED_TAG)).standard_normal((n, k))
    else:
        V = np.array(v0, dtype=np.float64)
    V /= np.linalg.norm(V, axis=0)
    best = 0.0
    for _ in range(iters):
        W = spmm(S, V)
        rq = np.einsum("ij,ij->j", V, W)
        best = max(best, float(np.max(np.abs(rq))))
        nrm = np.linalg.norm(W, axis=0)
        alive = nrm > 0.0
        if not np.any(alive):
            break
        V = W[:, alive] / nrm[alive]
    return best * safety


def norm_start_block(n: int, seed: int, factor: float = 6.0) -> np.ndarray:
    """The reference's PCG64 starting block (engine.py:178-180), unnormalised."""
    k = max(1, math.ceil(factor * math.log(max(n, 2))))
    return np.random.default_rng(fold_seed(seed, NORM_SEED_TAG)).standard_normal((n, k))


def row_normalize(E: np.ndarray) -> np.ndarray:
    """Row normalisation with zero rows -> 0 (semantics of oracle.py:88-96)."""
    E = np.asarray(E, dtype=np.float64)
    nr = np.linalg.norm(E, axis=1)
    out = np.zeros_like(E)
    nz = nr > 0
    out[nz] = E[nz] / nr[nz, None]
    return out


def pair_cosines(E: np.ndarray, pairs: np.ndarray) -> np.ndarray:
    """oracle._pair_correlations (oracle.py:88-96): cosine, zero rows give 0."""
    E = np.asarray(E, dtype=np.float64)
    nr = np.linalg.norm(E, axis=1)
    a, b = pairs[:, 0], pairs[:, 1]
    den = nr[a] * nr[b]
    dots = np.einsum("ij,ij->i", E[a], E[b])
    out = np.zeros(len(pairs))
    np.divide(dots, den, out=out, where=den != 0.0)
    return out


def sample_pairs(n: int, n_pairs: int, seed: int) -> np.ndarray:
    """oracle.sample_pairs (oracle.py:99-119): uniform i<j pairs w/o replacement."""
    total = n * (n - 1) // 2
    n_pairs = min(n_pairs, total)
    if n_pairs == total:
        return np.stack(np.triu_indices(n, k=1), axis=1).astype(np.int64)
    rng = np.random.default_rng(seed)
    codes = np.empty(0, dtype=np.uint64)
    while len(codes) < n_pairs:
        want = n_pairs - len(codes)
        i = rng.integers(0, n, size=2 * want + 16)
        j = rng.integers(0, n, size=2 * want + 16)
        ok = i != j
        lo = np.minimum(i[ok], j[ok]).astype(np.uint64)
        hi = np.maximum(i[ok], j[ok]).astype(np.uint64)
        codes = np.unique(np.concatenate([codes, lo * np.uint64(n) + hi]))
    codes = codes[:n_pairs]
    return np.stack([codes // np.uint64(n), codes % np.uint64(n)], axis=1).astype(np.int64)


# -- downstream consumers (reference cluster.py) ------------------------------


def _sqdist(X: np.ndarray, Cn: np.ndarray) -> np.ndarray:
    """cluster._sq_distances (cluster.py:34-40): max(|x|^2 + |c|^2 - 2 x.c, 0)."""
    g = X @ Cn.T
    return np.maximum(np.sum(X * X, axis=1)[:, None] + np.sum(Cn * Cn, axis=1)[None, :] - 2.0 * g, 0.0)


def kmeans(X: np.ndarray, K: int, max_iters: int = 100, seed: int = 0):
    """cluster.kmeans (cluster.py:43-107): k-means++ seeding then Lloyd
    iterations; returns (labels, inertia_history).  Same Generator draws:
    integers(n) for the first centroid and the zero-total branch, choice(n, p)
    for weighted picks; empty clusters take the farthest remaining point and
    skip the mean update; stop when labels repeat."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    if not 1 <= K <= n:
        raise ValueError(f"K={K} must lie in [1, n_rows={n}]")
    rng = np.random.default_rng(seed)
    cent = np.empty((K, X.shape[1]))
    cent[0] = X[rng.integers(n)]
    near = _sqdist(X, cent[:1])[:, 0]
    for k in range(1, K):
        tot = near.sum()
        row = int(rng.integers(n)) if tot <= 0.0 else int(rng.choice(n, p=near / tot))
        cent[k] = X[row]
        near = np.minimum(near, _sqdist(X, cent[k:k + 1])[:, 0])
    labels = np.full(n, -1, dtype=np.int64)
    hist: list[float] = []
    for _ in range(max_iters):
        d2 = _sqdist(X, cent)
        new = np.argmin(d2, axis=1).astype(np.int64)
        best = d2[np.arange(n), new]
        hist.append(float(best.sum()))
        sizes = np.bincount(new, minlength=K)
        if (sizes == 0).any():
            free = best.copy()
            for c in np.flatnonzero(sizes == 0):
                far = int(np.argmax(free))
                cent[c], new[far], free[far] = X[far], c, -1.0
            labels = new
            continue
        done = np.array_equal(new, labels)
        labels = new
        if done:
            break
        acc = np.zeros_like(cent)
        np.add.at(acc, labels, X)
        cent = acc / np.bincount(labels, minlength=K)[:, None]
    return labels, hist


def modularity(edges: np.ndarray, labels: np.ndarray) -> tuple[float, int]:
    """cluster.modularity (cluster.py:110-128) -> (Q, m) over the simple
    undirected graph of `edges` (loops dropped, duplicates merged)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    e = e[e[:, 0] != e[:, 1]]
    und = np.unique(np.sort(e, axis=1), axis=0)
    m = len(und)
    lab = np.asarray(labels, dtype=np.int64)
    k = int(lab.max()) + 1
    lu, lv = lab[und[:, 0]], lab[und[:, 1]]
    intra = np.bincount(lu[lu == lv], minlength=k)
    deg = np.bincount(und.ravel(), minlength=len(lab))
    degsum = np.bincount(lab, weights=deg, minlength=k)
    return float(np.sum(intra / m - (degsum / (2.0 * m)) ** 2)), m


__all__ = [
    "CSR", "build", "lib", "set_threads", "num_threads", "fold_seed", "sample_projection",
    "np_sample_projection", "spmm", "run_stage", "apply_expansion", "spectral_norm",
    "norm_start_block", "row_normalize", "pair_cosines", "sample_pairs", "NORM_SEED_TAG", "kmeans",
    "modularity",
]
