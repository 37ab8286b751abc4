"""Multi-GPU column sharding (one process per GPU, torch.distributed plumbing).

The d projection columns are independent (reference Theorem 1 / column-subset
bit-exactness, tests/test_engine.py:152-160), so each rank holds the whole
matrix and runs the fused recurrence on its own column slice [lo, hi) of the
n x d block -- hashed with the GLOBAL d (engine.py:96), so every entry of the
assembled E is bit-identical to the single-GPU result.  The only exchange is
one all-gather of the E slices (NCCL over NVLink on GPUs; gloo in the CPU
tests), after which E is row-normalised on the device.

Shard boundaries are multiples of the 16-byte vector width (2 columns in f64,
4 in f32) so a vector never straddles two ranks or two of the reference's
32-column diagnostic chunks.
"""

from __future__ import annotations

import numpy as np


def column_shards(d: int, world: int, align: int = 1) -> list[tuple[int, int]]:
    """Contiguous, as-balanced-as-possible slices of [0, d) whose boundaries
    are multiples of `align` (the last one ends at d)."""
    if d < 1 or world < 1 or align < 1:
        raise ValueError("d, world and align must be positive")
    cuts = [0]
    for r in range(1, world):
        c = int(round(d * r / world / align)) * align
        cuts.append(min(max(c, cuts[-1]), d))
    cuts.append(d)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def assemble_columns(local, world: int, d: int, dtype: str = "f64", group=None):
    """All-gather per-rank (n x w_r) column slices into the full (n x d) block.

    Uses torch.distributed.all_gather on slices padded to the widest shard
    (NCCL requires equal shapes), then drops the padding."""
    import torch
    import torch.distributed as dist

    align = 2 if dtype == "f64" else 4
    shards = column_shards(d, world, align)
    wmax = max(hi - lo for lo, hi in shards)
    n = local.shape[0]
    padded = local
    if local.shape[1] != wmax:
        padded = torch.zeros((n, wmax), dtype=local.dtype, device=local.device)
        padded[:, : local.shape[1]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded.contiguous(), group=group)
    return torch.cat([p[:, : hi - lo] for p, (lo, hi) in zip(parts, shards)], dim=1).contiguous()


def combine_peaks(peaks: np.ndarray, group=None) -> np.ndarray:
    """Max-combine per-chunk |Q(r)| keys across ranks (NaN/inf keys dominate,
    so divergence found on any rank is reported everywhere)."""
    import torch
    import torch.distributed as dist

    keys = torch.from_numpy(np.ascontiguousarray(peaks).view(np.int64).copy())
    if dist.get_backend(group) == "nccl":
        keys = keys.cuda()
    dist.all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
    return keys.cpu().numpy().view(np.float64).reshape(peaks.shape)


def embed_column_sharded(S, coeffs, d: int, *, n_stages: int = 1, seed: int = 0, omega_kind: str = "reference",
                         dtype: str = "f64", normalize_rows: bool = True, group=None, device: int | None = None,
                         compute=None):
    """E = f_L(S) Omega over `d` columns sharded across the ranks of `group`.

    `compute(lo, hi)` may replace the device recurrence (the CPU tests inject
    the oracle); by default each rank runs the fused CUDA path on its GPU.
    Returns the assembled (n x d) torch tensor on every rank and the combined
    per-chunk peaks."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .engine import _OMEGA, DeviceMatrix

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    align = 2 if dtype == "f64" else 4
    lo, hi = column_shards(d, world, align)[rank]
    if compute is not None:
        local, peaks = compute(lo, hi)
        E = assemble_columns(local, world, d, dtype, group)
        return E, combine_peaks(peaks, group)
    device = torch.cuda.current_device() if device is None else device
    dm = DeviceMatrix(S, "float64" if dtype == "f64" else "float32", device)
    plan = dm.plan(hi - lo)
    plan.run(coeffs, n_stages, omega_kind=_OMEGA[omega_kind], seed=seed, col0=lo, d_global=d)
    peaks, _, _ = plan.diagnostics()
    tdt = torch.float64 if dtype == "f64" else torch.float32
    local = torch.empty((S.n_rows, hi - lo), dtype=tdt, device=f"cuda:{device}")
    plan.copy_output_to(local.data_ptr(), hi - lo)
    dm.ctx.sync()
    E = assemble_columns(local, world, d, dtype, group)
    if normalize_rows:
        _lib.check(dm.lib.csemb_rownorm(dm.ctx.handle, E.data_ptr(), E.shape[0], d, d,
                                        _lib.F64 if dtype == "f64" else _lib.F32), "csemb_rownorm")
        dm.ctx.sync()
    dm.close()
    return E, combine_peaks(peaks, group)
