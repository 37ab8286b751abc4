"""Device-side input construction.

The reference builds its inputs on the host (sparse.py:191-226): dedupe the
undirected edge list, drop self-loops, degrees by bincount, values
1/sqrt(deg_u * deg_v) (`normalized_adjacency`), and the dilation
[0 A^T; A 0] (`dilate`).  At config-2..5 scale that host work dominates the
end-to-end time (20.5 s at n = 1e6), so the builders here run as this
package's own kernels behind the C ABI (csrc/build.cu:
csemb_build_normalized_adjacency / csemb_build_dilation): edge keys, radix
sort + unique, degree counts, scan, symmetric keys, radix sort, one fused
column/value pass.  The arithmetic is the reference's (same IEEE expression
per value) and the CSR is canonical (rows ascending, columns strictly
increasing), so it is bit-identical to the host builders
(tests/test_gpu_parity.py::TestDeviceBuild).

The results are `DeviceCSR` objects: the library-owned device matrix plus
zero-copy torch views of its arrays (int64 offsets, int32 columns, f64
values) for callers that slice or inspect them on the device.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .engine import DeviceMatrix, dtype_code

BUILDER_KIND = "csemb kernels (csrc/build.cu: keys, CUB radix sort/unique/scan, degree + fill kernels)"


class _DeviceArray:
    """__cuda_array_interface__ over a library-owned device array; torch keeps
    this object (and through it the owning matrix) alive with the tensor."""

    def __init__(self, ptr: int, n: int, typestr: str, owner):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": typestr,
                                         "strides": None, "version": 3, "stream": None}
        self._owner = owner


class DeviceCSR:
    """A canonical CSR on one GPU: int64 offsets, int64 or int32 columns, f64
    values as torch CUDA tensors (optionally views of a library matrix)."""

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values, owner: DeviceMatrix | None = None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_offsets, self.col_indices, self.values = row_offsets, col_indices, values
        self.owner = owner

    @classmethod
    def from_matrix(cls, dm: DeviceMatrix) -> "DeviceCSR":
        """Zero-copy views of a library matrix's arrays (f64 matrices)."""
        if dm.dtype != _lib.F64:
            raise ValueError("DeviceCSR views need an f64 matrix")
        ro, ci, va = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _lib.check(dm.lib.csemb_matrix_device_arrays(dm.handle, C.byref(ro), C.byref(ci), C.byref(va)),
                   "csemb_matrix_device_arrays")
        dev = torch.device("cuda", dm.ctx.device)

        def view(ptr, n, typestr, dt):
            if n == 0:
                return torch.empty(0, dtype=dt, device=dev)
            return torch.as_tensor(_DeviceArray(ptr.value, n, typestr, dm), device=dev)

        return cls(dm.n_rows, dm.n_cols, view(ro, dm.n_rows + 1, "<i8", torch.int64),
                   view(ci, dm.nnz, "<i4", torch.int32), view(va, dm.nnz, "<f8", torch.float64), owner=dm)

    @property
    def nnz(self) -> int:
        return int(self.values.numel())

    def to_device_matrix(self, dtype="float64", device: int | None = None) -> DeviceMatrix:
        dev = self.values.device.index if device is None else device
        if self.owner is not None and dev == self.owner.ctx.device:  # device-side copy in the requested dtype
            h = C.c_void_p()
            _lib.check(self.owner.lib.csemb_matrix_convert(self.owner.handle, dtype_code(dtype), C.byref(h)),
                       "csemb_matrix_convert")
            return DeviceMatrix(None, dtype, dev, _handle=h)
        ro, ci, va = self.row_offsets, self.col_indices, self.values
        if va.device.index != dev:  # the library's kernels read device-local arrays only
            ro, ci, va = (t.to(f"cuda:{dev}") for t in (ro, ci, va))
        # the tensors may still be in flight on torch's stream (NCCL broadcasts of
        # distributed.broadcast_matrix, builder kernels, the copy above): the
        # library stream must not read them before that work completes
        torch.cuda.current_stream(va.device).synchronize()
        return DeviceMatrix.from_device(self.n_rows, self.n_cols, self.nnz, ro.data_ptr(),
                                        ci.data_ptr(), ci.element_size(), va.data_ptr(), dtype, dev)

    def to_host(self):
        from .sparse import SparseMatrix

        return SparseMatrix(self.n_rows, self.n_cols, self.row_offsets.cpu().numpy(),
                            self.col_indices.cpu().numpy().astype("int64"), self.values.cpu().numpy(),
                            check=False)


def normalized_adjacency(edges, n: int, device: int | None = None) -> DeviceCSR:
    """D^{-1/2} A D^{-1/2} of the simple graph, built on the GPU by the
    library's kernels (sparse.py:202-226).  `edges`: (E, 2) int64, a CUDA
    tensor (read in place) or a host array (copied once)."""
    if n < 1:
        raise ValueError("vertex count must be positive")
    if isinstance(edges, torch.Tensor) and edges.is_cuda:
        e = edges.reshape(-1, 2).to(torch.int64).contiguous()
        dev = e.device.index if device is None else device
        torch.cuda.current_stream(e.device).synchronize()  # produced on torch's stream
        ptr, on_dev, n_edges = e.data_ptr(), 1, e.shape[0]
    else:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
        dev = 0 if device is None else device
        ptr, on_dev, n_edges = e.ctypes.data, 0, e.shape[0]
    ctx = _lib.context(dev)
    h = C.c_void_p()
    _lib.check(ctx.lib.csemb_build_normalized_adjacency(ctx.handle, int(n), int(n_edges), C.c_void_p(ptr),
                                                        on_dev, _lib.F64, C.byref(h)),
               "csemb_build_normalized_adjacency")
    return DeviceCSR.from_matrix(DeviceMatrix(None, "float64", dev, _handle=h))


def dilate(A: DeviceCSR) -> DeviceCSR:
    """[0 A^T; A 0] on the GPU: first n indices are A's columns, last m its rows
    (sparse.py:191-199), by the library's transpose + fill kernels."""
    if A.n_rows < 1 or A.n_cols < 1:
        raise ValueError("cannot dilate an empty matrix")
    src = A.owner if A.owner is not None else A.to_device_matrix("float64")
    h = C.c_void_p()
    _lib.check(src.lib.csemb_build_dilation(src.handle, C.byref(h)), "csemb_build_dilation")
    out = DeviceCSR.from_matrix(DeviceMatrix(None, "float64", src.ctx.device, _handle=h))
    if src is not A.owner:
        src.close()
    return out


def _offsets(rows: torch.Tensor, n_rows: int) -> torch.Tensor:
    """CSR offsets of sorted row ids (generators only)."""
    counts = torch.bincount(rows, minlength=n_rows)
    offs = torch.zeros(n_rows + 1, dtype=torch.int64, device=rows.device)
    torch.cumsum(counts, 0, out=offs[1:])
    return offs


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
