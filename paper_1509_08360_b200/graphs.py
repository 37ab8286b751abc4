"""Seeded O(T) synthetic inputs with the BASELINE configs' shapes.

The reference only ships an O(n^2) SBM test helper (tests/helpers.py:31-39),
so the benchmark-scale inputs are sampled here edge-by-edge:

  sbm_edges      config 2/5: planted partition, expected intra/inter degree
  chung_lu_edges config 3: Pareto(2.1) expected degrees in [2, 1e4], mean 20
  bag_of_words   config 4: Poisson(150) doc lengths, Zipf(1.1) term ids,
                 tf-idf counts, rows L2-normalised (rectangular m x n)

Graphs go through `normalized_adjacency` (dedupe, drop self-loops,
1/sqrt(deg u deg v)), exactly the reference's construction.  Everything is a
pure function of the seed (numpy PCG64).  These run on the host, outside
every timed region.
"""

from __future__ import annotations

import numpy as np

from .sparse import SparseMatrix, normalized_adjacency


def sbm_edges(n: int, blocks: int, deg_in: float, deg_out: float, seed: int) -> np.ndarray:
    """Planted partition with contiguous equal blocks; each intra edge joins a
    uniform vertex to a uniform vertex of its block, each inter edge to a
    uniform vertex of another block; E[intra degree] = deg_in, E[inter] = deg_out."""
    rng = np.random.default_rng(seed)
    bs = n // blocks
    m_in = int(round(n * deg_in / 2.0))
    m_out = int(round(n * deg_out / 2.0))
    u = rng.integers(0, n, size=m_in, dtype=np.int64)
    blk = np.minimum(u // bs, blocks - 1)
    lo = blk * bs
    size = np.where(blk == blocks - 1, n - lo, bs)
    v = lo + (rng.random(m_in) * size).astype(np.int64)
    u2 = rng.integers(0, n, size=m_out, dtype=np.int64)
    blk2 = np.minimum(u2 // bs, blocks - 1)
    lo2 = blk2 * bs
    size2 = np.where(blk2 == blocks - 1, n - lo2, bs)
    r = rng.integers(0, n, size=m_out, dtype=np.int64) % (n - size2)
    v2 = np.where(r >= lo2, r + size2, r)
    return np.stack([np.concatenate([u, u2]), np.concatenate([v, v2])], axis=1)


def sbm(n: int, blocks: int, deg_in: float, deg_out: float, seed: int) -> SparseMatrix:
    return normalized_adjacency(sbm_edges(n, blocks, deg_in, deg_out, seed), n)


def chung_lu_edges(n: int, seed: int, exponent: float = 2.1, w_min: float = 2.0, w_max: float = 1e4,
                   mean: float = 20.0) -> np.ndarray:
    """Chung-Lu with i.i.d. Pareto(exponent) weights clipped to [w_min, w_max]
    and rescaled to `mean`; edge (i, j) with p ~ w_i w_j / sum w, sampled in
    O(T) as sum(w)/2 endpoint pairs drawn proportional to w."""
    rng = np.random.default_rng(seed)
    w = w_min * (1.0 - rng.random(n)) ** (-1.0 / (exponent - 1.0))
    w = np.minimum(w, w_max)
    w *= mean / w.mean()
    m = int(round(w.sum() / 2.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = np.searchsorted(cdf, rng.random(m), side="right")
    v = np.searchsorted(cdf, rng.random(m), side="right")
    return np.stack([np.minimum(u, n - 1), np.minimum(v, n - 1)], axis=1).astype(np.int64)


def chung_lu(n: int, seed: int, **kw) -> SparseMatrix:
    return normalized_adjacency(chung_lu_edges(n, seed, **kw), n)


def bag_of_words(m: int, n: int, seed: int, mean_len: float = 150.0, zipf_s: float = 1.1) -> SparseMatrix:
    """m documents x n terms: Poisson(mean_len) tokens per document with
    Zipf(zipf_s) term ids truncated to n, tf-idf weighted counts
    (tf * log(m / df)), rows L2-normalised; empty rows stay empty."""
    rng = np.random.default_rng(seed)
    lens = rng.poisson(mean_len, size=m)
    tot = int(lens.sum())
    ranks = np.arange(1, n + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** (-zipf_s))
    cdf /= cdf[-1]
    terms = np.searchsorted(cdf, rng.random(tot), side="right").astype(np.int64)
    terms = np.minimum(terms, n - 1)
    docs = np.repeat(np.arange(m, dtype=np.int64), lens)
    key = np.unique(docs * n + terms, return_counts=True)
    keys, tf = key
    r, c = keys // n, keys % n
    df = np.bincount(c, minlength=n).astype(np.float64)
    idf = np.log(m / np.maximum(df, 1.0))
    vals = tf.astype(np.float64) * idf[c]
    keep = vals != 0.0
    r, c, vals = r[keep], c[keep], vals[keep]
    rn = np.sqrt(np.bincount(r, weights=vals * vals, minlength=m))
    vals = vals / rn[r]
    offs = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=m), out=offs[1:])
    return SparseMatrix(m, n, offs, c, vals, check=False)
