"""Sampled-pair correlation distortion with the pair work on the device
(reference oracle.py:88-275; SURVEY 8(d) parity harness and 8(f) rank 4).

``pair_correlations`` is ``_pair_correlations`` (oracle.py:88-96) on the GPU:
one K5 launch (csemb_pair_cosines) for any number of pairs, on a host block or
a device-resident embedding (DeviceRows, e.g. a plan's E -- no n x d
download).  Norms follow numpy's pairwise order exactly; the dot products use
the same order where the reference's einsum uses its own, so cosines agree to
a few ulps.  Pair sampling, percentiles, binning and report writers are host
code with the reference's exact numpy expressions.  ``exact_embedding`` (the
reference's desk-scale dense ground truth, oracle.py:29-71) runs the full
symmetric eigensolve on the device through cuSOLVER (torch.linalg.eigh, a
library call, not the hot path); pair correlations are invariant to the
eigensolver's sign and eigenspace-basis choices, so distortion reports match
the reference's to rounding.
"""

from __future__ import annotations

import csv
import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cluster import DeviceRows
from .engine import EmbeddingMatrix, apply_expansion, fold_seed, sample_projection
from .errors import OracleCapError, OracleError
from .legendre import expansion_eval, legendre_coefficients
from .sparse import SparseMatrix

ORACLE_CAP = 3000          # oracle.py:22
EIG_RESIDUAL_TOL = 1e-8   # oracle.py:23
PERCENTILE_LEVELS = (1, 5, 25, 50, 75, 95, 99)
DEFAULT_MAX_PAIRS = 100_000
CALIBRATION_BIN_WIDTH = 0.1  # bins centred on -1.0, -0.9, ..., 1.0


def sample_pairs(n: int, n_pairs: int | None, seed: int) -> np.ndarray:
    """Uniform vertex pairs (i < j) without replacement, deterministic per seed
    (oracle.py:99-119).  Same draw sequence as the reference: rounds of
    2*want+16 candidate (i, j) draws, self-pairs dropped, pairs encoded as
    lo*n + hi and merged through np.unique until enough are collected; the
    smallest n_pairs codes are kept.  Asking for every pair enumerates them."""
    n_all = n * (n - 1) // 2
    want_total = min(DEFAULT_MAX_PAIRS if n_pairs is None else n_pairs, n_all)
    if want_total == n_all:
        return np.column_stack(np.triu_indices(n, k=1)).astype(np.int64)
    rng = np.random.default_rng(seed)
    un = np.uint64(n)
    pool = np.empty(0, dtype=np.uint64)
    while pool.size < want_total:
        m = 2 * (want_total - pool.size) + 16
        a, b = rng.integers(0, n, size=m), rng.integers(0, n, size=m)
        keep = a != b
        a, b = a[keep], b[keep]
        fresh = np.minimum(a, b).astype(np.uint64) * un + np.maximum(a, b).astype(np.uint64)
        pool = np.unique(np.concatenate([pool, fresh]))
    pool = pool[:want_total]
    return np.column_stack([pool // un, pool % un]).astype(np.int64)


@dataclass
class ExactEmbedding:
    """Rows of f(S) in compact form: eigenvectors scaled by f(eigenvalue), exact
    zero weights dropped (oracle.py:29-43)."""

    embedding: np.ndarray
    eigenvalues: np.ndarray
    basis: str = "dense-eigh (cuSOLVER)"

    @property
    def n_rows(self) -> int:
        return self.embedding.shape[0]


def _dense_symmetric(S, cap: int) -> np.ndarray:
    a = S.to_dense() if isinstance(S, SparseMatrix) else np.asarray(S, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("expected a square matrix")
    if a.shape[0] > cap:
        raise OracleCapError(f"matrix of size {a.shape[0]} exceeds the dense-oracle cap {cap}")
    if np.max(np.abs(a - a.T), initial=0.0) > 1e-10:
        raise ValueError("oracle requires a symmetric matrix")
    return a


def _eigh_device(a: np.ndarray, device: int):
    """Full symmetric eigendecomposition on the GPU (cuSOLVER) with the
    reference's residual acceptance (oracle.py:58-63); host (lam, vec)."""
    import torch

    ta = torch.from_numpy(np.ascontiguousarray(a)).to(torch.device(f"cuda:{device}"))
    lam, vec = torch.linalg.eigh(ta)
    residual = float((ta @ vec - vec * lam).abs().max()) if a.size else 0.0
    if residual > EIG_RESIDUAL_TOL:
        raise OracleError(f"eigensolver residual {residual:.3e} above {EIG_RESIDUAL_TOL}")
    return lam.cpu().numpy(), vec.cpu().numpy()


def _pairwise_distances(rows: np.ndarray, device: int) -> np.ndarray:
    """Upper-triangle pairwise Euclidean distances, the reference's formula
    sqrt(max(|x|^2 + |y|^2 - 2 x.y, 0)) (oracle.py:219-224), in fp64 on the GPU."""
    import torch

    x = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float64)).to(torch.device(f"cuda:{device}"))
    sq = (x * x).sum(dim=1)
    d2 = sq[:, None] + sq[None, :] - 2.0 * (x @ x.T)
    iu = torch.triu_indices(x.shape[0], x.shape[0], offset=1, device=x.device)
    return torch.sqrt(torch.clamp(d2[iu[0], iu[1]], min=0.0))


def distance_bound_audit(S, f, cfg, trials: int, cap: int = ORACLE_CAP, *, device: int = 0) -> float:
    """Fraction of (trial, pair) events violating the two-sided distance bound
    sqrt(1 -+ eps) * (exact distance -+ delta sqrt(2)) (oracle.py:196-216), where
    delta is the expansion's worst error at the true eigenvalues.  Each trial
    draws a fresh projection (the reference's hash, bit-identical) and embeds
    through the device seam; exact spectrum and distances on the GPU."""
    import math

    import torch

    a = _dense_symmetric(S, cap)
    lam, vec = _eigh_device(a, device)
    weights = np.atleast_1d(np.asarray(f(lam), dtype=np.float64))
    expansion = legendre_coefficients(f, cfg.L)
    delta = float(np.max(np.abs(weights - expansion_eval(expansion, lam)), initial=0.0))
    d_exact = _pairwise_distances(vec * weights, device)
    slack = delta * math.sqrt(2.0)
    lower = math.sqrt(1.0 - cfg.epsilon) * (d_exact - slack)
    upper = math.sqrt(1.0 + cfg.epsilon) * (d_exact + slack)
    sp = SparseMatrix.from_dense(a)
    n = a.shape[0]
    violations = 0
    for t in range(trials):
        omega = sample_projection(n, cfg.d, fold_seed(cfg.seed, t), device=device)
        emb = apply_expansion(sp, expansion, omega, device=device)
        d_approx = _pairwise_distances(emb, device)
        violations += int(torch.count_nonzero((d_approx < lower) | (d_approx > upper)))
    return violations / (trials * d_exact.numel())


def exact_embedding(S, f, cap: int = ORACLE_CAP, *, device: int = 0) -> ExactEmbedding:
    """Exact embedding by a full dense symmetric eigendecomposition on the GPU
    (oracle.py:46-71 semantics: square and symmetric to 1e-10, at most `cap`
    rows, eigen-residual <= 1e-8, weights f(lambda), zero weights dropped)."""
    a = _dense_symmetric(S, cap)
    lam, vec = _eigh_device(a, device)
    weights = np.atleast_1d(np.asarray(f(lam), dtype=np.float64))
    keep = weights != 0.0
    return ExactEmbedding(embedding=vec[:, keep] * weights[keep], eigenvalues=lam)


def _rows(x):
    if isinstance(x, DeviceRows):
        return x
    if isinstance(x, EmbeddingMatrix):
        x = x.values
    x = getattr(x, "embedding", x)  # the reference's ExactEmbedding
    a = np.asarray(x)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-d block of rows")
    return np.ascontiguousarray(a)


def _n_rows(x) -> int:
    return x.n if isinstance(x, DeviceRows) else x.shape[0]


def pair_correlations(rows, pairs, *, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """(cosine per pair, zero-norm flag per pair) -- _pair_correlations on the GPU."""
    rows = _rows(rows)
    pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
    out = np.zeros(len(pairs))
    zero = np.zeros(len(pairs), dtype=np.uint8)
    if isinstance(rows, DeviceRows):
        ctx = _lib.context(rows.device)
        rc = ctx.lib.csemb_pair_cosines(ctx.handle, C.c_void_p(rows.ptr), rows.dtype, 1, rows.n, rows.d, rows.ld,
                                        _lib.ptr(pairs), len(pairs), _lib.ptr(out), _lib.ptr(zero))
    else:
        ctx = _lib.context(device)
        code = _lib.F64 if rows.dtype == np.float64 else _lib.F32
        n, d = rows.shape
        rc = ctx.lib.csemb_pair_cosines(ctx.handle, _lib.ptr(rows), code, 0, n, d, d, _lib.ptr(pairs), len(pairs),
                                        _lib.ptr(out), _lib.ptr(zero))
    _lib.check(rc, "csemb_pair_cosines")
    return out, zero.astype(bool)


def normalized_correlation(X, i: int, j: int, *, device: int = 0) -> float:
    """Cosine similarity of rows i and j; zero rows correlate as 0 (oracle.py:79-85)."""
    return float(pair_correlations(X, np.array([[i, j]]), device=device)[0][0])


@dataclass
class CalibrationBin:
    center: float
    count: int
    percentiles: dict[int, float]


@dataclass
class DistortionReport:
    """Percentiles of correlation deviation, or per-bin calibration curves."""

    mode: str
    pair_sample_size: int
    zero_row_pairs: int = 0
    percentiles: dict[int, float] | None = None
    bins: list[CalibrationBin] = field(default_factory=list)


def _pct(values) -> dict[int, float]:
    return dict(zip(PERCENTILE_LEVELS, (float(v) for v in np.percentile(values, PERCENTILE_LEVELS))))


def _calibration_bins(exact_corr: np.ndarray, approx_corr: np.ndarray) -> list[CalibrationBin]:
    """Bins of width 0.1 centred on -1.0 .. 1.0 by exact correlation (rounded
    to the nearest centre, clipped); empty bins are omitted (oracle.py:166-181)."""
    centres = np.round(np.arange(-1.0, 1.0 + CALIBRATION_BIN_WIDTH / 2, CALIBRATION_BIN_WIDTH), 10)
    slot = np.clip(np.round((exact_corr + 1.0) / CALIBRATION_BIN_WIDTH).astype(int), 0, len(centres) - 1)
    out = []
    for b, centre in enumerate(centres):
        members = approx_corr[slot == b]
        if members.size:
            out.append(CalibrationBin(center=float(centre), count=int(members.size), percentiles=_pct(members)))
    return out


def distortion_percentiles(exact, approx, n_pairs: int | None = None, seed: int = 0, mode: str = "deviation",
                           *, device: int = 0) -> DistortionReport:
    """Compare normalized correlations of two embeddings over sampled pairs
    (oracle.py:139-186): ``deviation`` reports percentiles of approx - exact;
    ``calibration`` bins pairs by exact correlation and reports percentiles
    of the approximate correlation per bin.  Both correlation passes are
    single device launches."""
    X, Y = _rows(exact), _rows(approx)
    if _n_rows(X) != _n_rows(Y):
        raise ValueError("embeddings must have the same number of rows")
    if mode not in ("deviation", "calibration"):
        raise ValueError("mode must be 'deviation' or 'calibration'")
    pairs = sample_pairs(_n_rows(X), n_pairs, seed)
    cx, zx = pair_correlations(X, pairs, device=device)
    cy, zy = pair_correlations(Y, pairs, device=device)
    report = DistortionReport(mode=mode, pair_sample_size=len(pairs), zero_row_pairs=int(np.count_nonzero(zx | zy)))
    if mode == "deviation":
        report.percentiles = _pct(cy - cx)
    else:
        report.bins = _calibration_bins(cx, cy)
    return report


# -- report serialization (formats of oracle.py:227-275) ---------------------


def report_to_dict(report: DistortionReport) -> dict:
    doc = {"mode": report.mode, "pair_sample_size": report.pair_sample_size,
           "zero_row_pairs": report.zero_row_pairs}
    if report.percentiles is not None:
        doc["percentiles"] = {str(level): v for level, v in report.percentiles.items()}
    if report.bins:
        doc["bins"] = [{"center": b.center, "count": b.count,
                        "percentiles": {str(level): v for level, v in b.percentiles.items()}}
                       for b in report.bins]
    return doc


def _write_csv(path, header, rows) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)


def write_percentiles_csv(report: DistortionReport, path) -> None:
    if report.percentiles is None:
        raise ValueError("report has no deviation percentiles")
    _write_csv(path, ["percentile", "value"], ([p, repr(report.percentiles[p])] for p in PERCENTILE_LEVELS))


def write_calibration_csv(report: DistortionReport, path) -> None:
    if not report.bins:
        raise ValueError("report has no calibration bins")
    _write_csv(path, ["bin_center"] + [f"p{p}" for p in PERCENTILE_LEVELS],
               ([b.center] + [repr(b.percentiles[p]) for p in PERCENTILE_LEVELS] for b in report.bins))


def write_report_json(report: DistortionReport, path) -> None:
    with open(path, "w") as fh:
        json.dump(report_to_dict(report), fh, indent=2, sort_keys=True)
        fh.write("\n")
