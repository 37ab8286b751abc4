"""Downstream validation on the device: k-means on embedding rows, scored by
graph modularity (reference cluster.py:1-171).

The host side replays the reference's control flow and its numpy Generator
draw sequence exactly (``rng.integers(n)`` for the first centroid and the
``total <= 0`` branch, one ``rng.random()`` per weighted pick -- what
``rng.choice(n, p=...)`` consumes); everything that touches the n x d rows
runs on the GPU through the C ABI (csemb_kmeans_*, csemb_modularity_counts):
distances, the weighted pick, the assignment GEMM + argmin, empty-cluster
re-seeding, centroid means and the modularity counts.

Arithmetic: squared norms and dot products follow numpy's pairwise order with
separately rounded products, and centroid sums follow np.add.at's row order,
so for the same labels the centroids are bit-identical to the reference; the
reference's X @ C.T comes from BLAS (unspecified order), so distances agree to
a few ulps and labels agree except at exact-tie distances.  Modularity is
formed from exact integer counts with the reference's own numpy expression.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import DeviceMatrix, EmbedConfig, EmbeddingMatrix, device_matrix, fast_embed_cascaded, fold_seed
from .sparse import normalized_adjacency, simple_edges

_KMEANS_SEED_TAG = 0x6B6D6531  # cluster.py:12, distinct stream from projection sampling


@dataclass
class ClusterAssignment:
    labels: np.ndarray
    K: int
    inertia: float
    n_iters: int = 0
    inertia_history: tuple[float, ...] = ()


@dataclass
class ModularityScore:
    Q: float
    m_edges: int

    def __post_init__(self):
        if not -0.5 - 1e-9 <= self.Q <= 1.0 + 1e-9:
            raise ValueError(f"modularity {self.Q} outside [-0.5, 1]")


@dataclass
class DeviceRows:
    """An n x d row block already in device memory (e.g. a plan's E)."""

    ptr: int
    n: int
    d: int
    ld: int
    dtype: int = _lib.F64
    device: int = 0
    owner: object = field(default=None, repr=False)  # keeps the buffer alive


def plan_rows(plan) -> DeviceRows:
    """The device-resident embedding of a finished plan run."""
    p, ld, dt = plan.output()
    return DeviceRows(p, plan.dm.n_rows, plan.d, ld, dt, plan.dm.ctx.device, plan)


def _host_rows(X) -> np.ndarray:
    rows = X.values if isinstance(X, EmbeddingMatrix) else getattr(X, "embedding", X)
    rows = np.asarray(rows, dtype=np.float64)
    if rows.ndim != 2:
        raise ValueError("expected a 2-d block of rows")
    return np.ascontiguousarray(rows)


class DeviceKMeans:
    """A csemb_kmeans handle: an f64 device copy of the rows plus Lloyd state."""

    def __init__(self, X, K: int, device: int = 0):
        if isinstance(X, DeviceRows):
            device = X.device
        self.ctx = _lib.context(device)
        self.lib = self.ctx.lib
        h = C.c_void_p()
        if isinstance(X, DeviceRows):
            self.n, self.d = X.n, X.d
            rc = self.lib.csemb_kmeans_create(self.ctx.handle, C.c_void_p(X.ptr), X.dtype, 1, X.n, X.d, X.ld,
                                              int(K), C.byref(h))
        else:
            rows = _host_rows(X)
            self.n, self.d = rows.shape
            rc = self.lib.csemb_kmeans_create(self.ctx.handle, _lib.ptr(rows), _lib.F64, 0, self.n, self.d,
                                              self.d, int(K), C.byref(h))
        _lib.check(rc, "csemb_kmeans_create")
        self.handle = h
        self.K = int(K)

    def reset(self) -> None:
        _lib.check(self.lib.csemb_kmeans_reset(self.handle), "csemb_kmeans_reset")

    def seed(self, k: int, row: int) -> float:
        total = C.c_double()
        _lib.check(self.lib.csemb_kmeans_seed(self.handle, int(k), int(row), C.byref(total)), "csemb_kmeans_seed")
        return float(total.value)

    def pick(self, u: float) -> int:
        row = C.c_int64()
        _lib.check(self.lib.csemb_kmeans_pick(self.handle, float(u), C.byref(row)), "csemb_kmeans_pick")
        return int(row.value)

    def assign(self) -> tuple[float, int, np.ndarray]:
        inertia, changed = C.c_double(), C.c_int64()
        counts = np.zeros(self.K, dtype=np.int64)
        _lib.check(self.lib.csemb_kmeans_assign(self.handle, C.byref(inertia), C.byref(changed), _lib.ptr(counts)),
                   "csemb_kmeans_assign")
        return float(inertia.value), int(changed.value), counts

    def reseed(self, c: int) -> int:
        row = C.c_int64()
        _lib.check(self.lib.csemb_kmeans_reseed(self.handle, int(c), C.byref(row)), "csemb_kmeans_reseed")
        return int(row.value)

    def commit(self, update_centroids: bool) -> None:
        _lib.check(self.lib.csemb_kmeans_commit(self.handle, int(bool(update_centroids))), "csemb_kmeans_commit")

    def labels(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int64)
        _lib.check(self.lib.csemb_kmeans_download(self.handle, _lib.ptr(out), None), "csemb_kmeans_download")
        return out

    def centroids(self) -> np.ndarray:
        out = np.empty((self.K, self.d), dtype=np.float64)
        _lib.check(self.lib.csemb_kmeans_download(self.handle, None, _lib.ptr(out)), "csemb_kmeans_download")
        return out

    def set_centroids(self, centroids) -> None:
        c = np.ascontiguousarray(centroids, dtype=np.float64)
        if c.shape != (self.K, self.d):
            raise ValueError(f"centroids must be {self.K} x {self.d}")
        _lib.check(self.lib.csemb_kmeans_set_centroids(self.handle, _lib.ptr(c)), "csemb_kmeans_set_centroids")

    def labels_device(self) -> int:
        return int(self.lib.csemb_kmeans_labels(self.handle) or 0)

    def close(self) -> None:
        if self.handle:
            self.lib.csemb_kmeans_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _run_kmeans(km: DeviceKMeans, K: int, max_iters: int, seed: int) -> ClusterAssignment:
    """The reference's loop (cluster.py:69-107) over the device steps."""
    n = km.n
    rng = np.random.default_rng(seed)
    # _plus_plus_init (cluster.py:43-56)
    total = km.seed(0, int(rng.integers(n)))
    for k in range(1, K):
        if total <= 0.0:
            pick = int(rng.integers(n))
        else:
            if not np.isfinite(total):  # rng.choice rejects such weights before drawing
                raise ValueError("Probabilities contain NaN")
            pick = km.pick(float(rng.random()))  # == rng.choice(n, p=closest / total)
        total = km.seed(k, pick)
    history: list[float] = []
    for _ in range(1, max_iters + 1):
        inertia, changed, counts = km.assign()
        if history and inertia > history[-1] * (1.0 + 1e-9) + 1e-12:
            raise RuntimeError("k-means inertia increased; numerical invariant broken")
        history.append(inertia)
        empties = np.flatnonzero(counts == 0)
        if len(empties):
            for c in empties:
                km.reseed(int(c))
            km.commit(False)
            continue
        converged = changed == 0
        km.commit(not converged)  # labels = new_labels; means unless converged
        if converged:
            break
    return ClusterAssignment(labels=km.labels(), K=K, inertia=history[-1], n_iters=len(history),
                             inertia_history=tuple(history))


def kmeans(X, K: int, max_iters: int = 100, seed: int = 0, *, device: int = 0,
           handle: DeviceKMeans | None = None) -> ClusterAssignment:
    """Lloyd iterations with distance-weighted seeding, deterministic per seed
    (cluster.py:59-107), on the device.  X: rows (ndarray / EmbeddingMatrix /
    DeviceRows).  ``handle`` reuses a DeviceKMeans built on the same rows."""
    if handle is None:
        n = X.n if isinstance(X, DeviceRows) else _host_rows(X).shape[0]
        if not 1 <= K <= n:
            raise ValueError(f"K={K} must lie in [1, n_rows={n}]")
        km = DeviceKMeans(X, K, device)
        try:
            return _run_kmeans(km, K, max_iters, seed)
        finally:
            km.close()
    if handle.K != K:
        raise ValueError("handle was built for a different K")
    handle.reset()
    return _run_kmeans(handle, K, max_iters, seed)


def _score(intra: np.ndarray, degsum: np.ndarray, m: int) -> ModularityScore:
    # cluster.py:127 with intra int64 and degsum float64, exactly as bincount returns them
    q = float(np.sum(intra / m - (degsum / (2.0 * m)) ** 2))
    return ModularityScore(Q=q, m_edges=m)


def modularity_counts(S, labels, k: int, *, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """(intra, degsum) per cluster from the CSR pattern of S (the simple
    undirected graph, each edge stored both ways).  labels: host array or a
    device pointer (int32) such as DeviceKMeans.labels_device()."""
    dm = S if isinstance(S, DeviceMatrix) else device_matrix(S, "float64", device)
    intra = np.zeros(k, dtype=np.int64)
    deg = np.zeros(k, dtype=np.int64)
    if isinstance(labels, int):
        rc = dm.lib.csemb_modularity_counts(dm.handle, C.c_void_p(labels), 1, int(k), _lib.ptr(intra), _lib.ptr(deg))
    else:
        lab = np.asarray(labels, dtype=np.int64)
        if len(lab) != dm.n_rows:
            raise ValueError("labels must cover all vertices")
        if lab.min(initial=0) < 0 or lab.max(initial=0) > np.iinfo(np.int32).max:
            raise ValueError("labels must be non-negative")
        lab32 = np.ascontiguousarray(lab, dtype=np.int32)
        rc = dm.lib.csemb_modularity_counts(dm.handle, _lib.ptr(lab32), 0, int(k), _lib.ptr(intra), _lib.ptr(deg))
    _lib.check(rc, "csemb_modularity_counts")
    return intra, deg.astype(np.float64)


def modularity(edges, labels, *, device: int = 0) -> ModularityScore:
    """Newman modularity Q = sum_c (intra_c / m - (degsum_c / 2m)^2) of an
    undirected simple graph under a vertex labeling (cluster.py:110-128)."""
    if isinstance(labels, ClusterAssignment) or hasattr(labels, "inertia_history"):
        labels = labels.labels
    labels = np.asarray(labels, dtype=np.int64)
    und = simple_edges(edges)
    m = len(und)
    if m == 0:
        raise ValueError("modularity needs at least one edge")
    if und.max() >= len(labels):
        raise ValueError("labels must cover all vertices")
    k = int(labels.max()) + 1
    pattern = normalized_adjacency(und, len(labels))  # CSR of the simple graph (values unused)
    dm = DeviceMatrix(pattern, "float32", device)
    try:
        intra, degsum = modularity_counts(dm, labels, k)
    finally:
        dm.close()
    return _score(intra, degsum, m)


@dataclass
class ClusterExperiment:
    median_modularity: float
    run_scores: tuple[float, ...]
    median_labels: np.ndarray
    embedding: EmbeddingMatrix = field(repr=False, default=None)


def cluster_experiment(edges, n: int, f, cfg: EmbedConfig, K: int, runs: int = 25, n_workers: int = 1, *,
                       dtype="float64", device: int = 0) -> ClusterExperiment:
    """Embed the graph's normalized adjacency compressively, then score ``runs``
    seeded K-means restarts by modularity and report the median
    (cluster.py:139-171).  The embedding, the restarts and the modularity
    counts stay on the device: one upload of the graph, no n x d round trip."""
    if runs < 1:
        raise ValueError("runs must be >= 1")
    adj = normalized_adjacency(edges, n)
    emb = fast_embed_cascaded(adj, f, cfg, n_workers=n_workers, dtype=dtype, device=device)
    m = adj.nnz // 2  # the simple edges of `edges` (normalized_adjacency's pattern)
    if m == 0:
        raise ValueError("modularity needs at least one edge")
    dm = device_matrix(adj, dtype, device)
    rows = plan_rows(dm.plan(emb.d))
    if not 1 <= K <= rows.n:
        raise ValueError(f"K={K} must lie in [1, n_rows={rows.n}]")
    km = DeviceKMeans(rows, K)
    scores, assignments = [], []
    try:
        for run in range(runs):
            a = kmeans(rows, K, seed=fold_seed(cfg.seed, _KMEANS_SEED_TAG + run), handle=km)
            k = int(a.labels.max()) + 1
            intra, degsum = modularity_counts(dm, km.labels_device(), k)
            scores.append(_score(intra, degsum, m).Q)
            assignments.append(a)
    finally:
        km.close()
    order = np.argsort(scores, kind="stable")
    median_idx = int(order[(runs - 1) // 2]) if runs % 2 else int(order[runs // 2 - 1])
    return ClusterExperiment(
        median_modularity=float(np.median(scores)),
        run_scores=tuple(scores),
        median_labels=assignments[median_idx].labels,
        embedding=emb,
    )
