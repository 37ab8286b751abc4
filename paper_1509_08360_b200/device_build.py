"""Device-side input construction.

The reference builds its inputs on the host (sparse.py:191-226): dedupe the
undirected edge list, drop self-loops, degrees by bincount, values
1/sqrt(deg_u * deg_v) (`normalized_adjacency`), and the dilation
[0 A^T; A 0] (`dilate`).  At config-3/4 scale (1e8 edges, 3e8 tokens) that
host work dominates the end-to-end time, so these builders do the same
construction on the GPU and hand the CSR to the C ABI without a host round
trip (`csemb_matrix_upload_device`).  Sorting/dedupe use torch's CUDA sort as
plumbing; the arithmetic is the reference's (same IEEE expression per
value), and the resulting CSR is canonical (rows ascending, columns strictly
increasing), so it is bit-identical to the host builders (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import torch

from .engine import DeviceMatrix


class DeviceCSR:
    """A canonical CSR held in torch CUDA tensors (int64 offsets, int64 or
    int32 columns, f64 values)."""

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_offsets, self.col_indices, self.values = row_offsets, col_indices, values

    @property
    def nnz(self) -> int:
        return int(self.values.numel())

    def to_device_matrix(self, dtype="float64", device: int | None = None) -> DeviceMatrix:
        dev = self.values.device.index if device is None else device
        ci = self.col_indices
        # the tensors may still be in flight on torch's stream (NCCL broadcasts of
        # distributed.broadcast_matrix, builder kernels): the library stream must
        # not read them before that work completes
        torch.cuda.current_stream(self.values.device).synchronize()
        return DeviceMatrix.from_device(self.n_rows, self.n_cols, self.nnz, self.row_offsets.data_ptr(),
                                        ci.data_ptr(), ci.element_size(), self.values.data_ptr(), dtype, dev)

    def to_host(self):
        from .sparse import SparseMatrix

        return SparseMatrix(self.n_rows, self.n_cols, self.row_offsets.cpu().numpy(),
                            self.col_indices.cpu().numpy().astype("int64"), self.values.cpu().numpy(),
                            check=False)


def _offsets(rows: torch.Tensor, n_rows: int) -> torch.Tensor:
    counts = torch.bincount(rows, minlength=n_rows)
    offs = torch.zeros(n_rows + 1, dtype=torch.int64, device=rows.device)
    torch.cumsum(counts, 0, out=offs[1:])
    return offs


def normalized_adjacency(edges: torch.Tensor, n: int) -> DeviceCSR:
    """D^{-1/2} A D^{-1/2} of the simple graph on the GPU (sparse.py:202-226)."""
    if n < 1:
        raise ValueError("vertex count must be positive")
    e = edges.reshape(-1, 2).to(torch.int64)
    if e.numel() and (int(e.min()) < 0 or int(e.max()) >= n):
        raise ValueError("edge endpoint out of range [0, n)")
    u, v = e[:, 0], e[:, 1]
    keep = u != v
    u, v = u[keep], v[keep]
    dev = e.device
    if u.numel() == 0:
        z = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        return DeviceCSR(n, n, z, torch.empty(0, dtype=torch.int32, device=dev),
                         torch.empty(0, dtype=torch.float64, device=dev))
    key = torch.unique(torch.minimum(u, v) * n + torch.maximum(u, v))  # sorted, deduped
    lo, hi = key // n, key % n
    del key
    deg = (torch.bincount(lo, minlength=n) + torch.bincount(hi, minlength=n)).to(torch.float64)
    sym = torch.cat([lo * n + hi, hi * n + lo])
    del lo, hi
    sym, _ = torch.sort(sym)
    r, c = sym // n, sym % n
    del sym
    vals = 1.0 / torch.sqrt(deg[r] * deg[c])  # same IEEE expression as the reference
    return DeviceCSR(n, n, _offsets(r, n), c.to(torch.int32), vals)


def dilate(A: DeviceCSR) -> DeviceCSR:
    """[0 A^T; A 0] on the GPU: first n indices are A's columns, last m its rows
    (sparse.py:191-199)."""
    m, n = A.n_rows, A.n_cols
    if m < 1 or n < 1:
        raise ValueError("cannot dilate an empty matrix")
    N = m + n
    dev = A.values.device
    r = torch.repeat_interleave(torch.arange(m, device=dev, dtype=torch.int64),
                                A.row_offsets[1:] - A.row_offsets[:-1])
    c = A.col_indices.to(torch.int64)
    keys = torch.cat([c * N + (n + r), (n + r) * N + c])
    vals = torch.cat([A.values, A.values])
    del r, c
    keys, order = torch.sort(keys, stable=True)
    vals = vals[order]
    rows = keys // N
    return DeviceCSR(N, N, _offsets(rows, N), (keys - rows * N).to(torch.int32), vals)


def from_host(S, device: int = 0) -> DeviceCSR:
    """Upload a host CSR into torch CUDA tensors."""
    d = torch.device(f"cuda:{device}")
    return DeviceCSR(S.n_rows, S.n_cols, torch.tensor(S.row_offsets, device=d),
                     torch.tensor(S.col_indices, device=d).to(torch.int32),
                     torch.tensor(S.values, device=d))


# -- seeded generators for configs 2-5 at full scale ---------------
def sbm_edges(n: int, blocks: int, deg_in: float, deg_out: float, seed: int, device: int = 0) -> torch.Tensor:
    """Configs 2 / 5 on the GPU: the planted partition of graphs.sbm_edges
    (contiguous equal blocks; each intra edge joins a uniform vertex to a
    uniform vertex of its block, each inter edge to a uniform vertex of another
    block), drawn with torch's CUDA generator."""
    dev = torch.device(f"cuda:{device}")
    g = torch.Generator(device=dev).manual_seed(seed)
    bs = n // blocks
    m_in, m_out = int(round(n * deg_in / 2.0)), int(round(n * deg_out / 2.0))
    out = torch.empty((m_in + m_out, 2), dtype=torch.int64, device=dev)
    u = torch.randint(0, n, (m_in,), generator=g, device=dev)
    blk = torch.clamp(u // bs, max=blocks - 1)
    lo = blk * bs
    size = torch.where(blk == blocks - 1, n - lo, torch.full_like(lo, bs))
    out[:m_in, 0] = u
    out[:m_in, 1] = lo + (torch.rand(m_in, generator=g, device=dev, dtype=torch.float64) * size).to(torch.int64)
    del u, blk, lo, size
    u2 = torch.randint(0, n, (m_out,), generator=g, device=dev)
    blk2 = torch.clamp(u2 // bs, max=blocks - 1)
    lo2 = blk2 * bs
    size2 = torch.where(blk2 == blocks - 1, n - lo2, torch.full_like(lo2, bs))
    r = torch.randint(0, n, (m_out,), generator=g, device=dev) % (n - size2)
    out[m_in:, 0] = u2
    out[m_in:, 1] = torch.where(r >= lo2, r + size2, r)
    return out



def chung_lu_edges(n: int, seed: int, device: int = 0, exponent: float = 2.1, w_min: float = 2.0,
                   w_max: float = 1e4, mean: float = 20.0) -> torch.Tensor:
    """Config 3: Pareto(exponent) expected degrees in [w_min, w_max], rescaled
    to `mean`; sum(w)/2 endpoint pairs drawn proportional to w (Chung-Lu)."""
    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed)
    dev = torch.device(f"cuda:{device}")
    u01 = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    w = w_min * (1.0 - u01) ** (-1.0 / (exponent - 1.0))
    w = torch.clamp(w, max=w_max)
    w *= mean / w.mean()
    m = int(round(float(w.sum()) / 2.0))
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    out = torch.empty((m, 2), dtype=torch.int64, device=dev)
    chunk = 1 << 26
    for lo in range(0, m, chunk):
        k = min(chunk, m - lo)
        for col in range(2):
            x = torch.rand(k, generator=g, device=dev, dtype=torch.float64)
            out[lo:lo + k, col] = torch.clamp(torch.searchsorted(cdf, x, right=True), max=n - 1)
    return out


def bag_of_words(m: int, n: int, seed: int, device: int = 0, mean_len: float = 150.0,
                 zipf_s: float = 1.1) -> DeviceCSR:
    """Config 4: m documents x n terms, Poisson(mean_len) tokens per document,
    Zipf(zipf_s) term ids truncated to n, tf * log(m/df) weights, rows
    L2-normalised."""
    dev = torch.device(f"cuda:{device}")
    g = torch.Generator(device=dev).manual_seed(seed)
    lens = torch.poisson(torch.full((m,), mean_len, device=dev, dtype=torch.float64), generator=g).to(torch.int64)
    cdf = torch.cumsum(torch.arange(1, n + 1, device=dev, dtype=torch.float64) ** (-zipf_s), 0)
    cdf /= cdf[-1].clone()
    docs = torch.repeat_interleave(torch.arange(m, device=dev, dtype=torch.int64), lens)
    tot = docs.numel()
    keys = torch.empty(tot, dtype=torch.int64, device=dev)
    chunk = 1 << 26
    for lo in range(0, tot, chunk):
        k = min(chunk, tot - lo)
        x = torch.rand(k, generator=g, device=dev, dtype=torch.float64)
        t = torch.clamp(torch.searchsorted(cdf, x, right=True), max=n - 1)
        keys[lo:lo + k] = docs[lo:lo + k] * n + t
    del docs
    keys, tf = torch.unique(keys, return_counts=True)
    r, c = keys // n, keys % n
    del keys
    df = torch.bincount(c, minlength=n).to(torch.float64)
    idf = torch.log(m / torch.clamp(df, min=1.0))
    vals = tf.to(torch.float64) * idf[c]
    keep = vals != 0.0
    r, c, vals = r[keep], c[keep], vals[keep]
    rn = torch.sqrt(torch.zeros(m, dtype=torch.float64, device=dev).index_add_(0, r, vals * vals))
    vals = vals / rn[r]
    return DeviceCSR(m, n, _offsets(r, m), c.to(torch.int32), vals)
