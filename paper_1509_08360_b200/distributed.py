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

import warnings

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


def broadcast_matrix(S, src: int = 0, group=None, device: int | None = None):
    """C1: replicate rank `src`'s CSR on every rank of `group`.

    Only `src` needs S (other ranks pass None).  The offsets (int64), column
    ids (int32) and values (f64) travel as three broadcasts: NCCL over NVLink
    for GPU tensors, landing directly in device memory as a DeviceCSR (upload
    with `.to_device_matrix`, no host copy); gloo on CPU returns a host
    SparseMatrix.  Values are bit-identical on every rank."""
    import torch
    import torch.distributed as dist

    from .sparse import SparseMatrix

    rank = dist.get_rank(group)
    on_gpu = dist.get_backend(group) == "nccl"
    dev = torch.device(f"cuda:{torch.cuda.current_device() if device is None else device}") if on_gpu \
        else torch.device("cpu")
    if rank == src:
        S = SparseMatrix.of(S)
        if S.n_cols > 0x7FFFFFFF:
            raise ValueError("column ids must fit in int32")
        meta = torch.tensor([S.n_rows, S.n_cols, S.nnz], dtype=torch.int64, device=dev)
        with warnings.catch_warnings():  # read-only (immutable) arrays: only ever copied out
            warnings.simplefilter("ignore", UserWarning)
            ro = torch.from_numpy(S.row_offsets).to(dev)
            ci = torch.from_numpy(S.col_indices.astype(np.int32)).to(dev)
            va = torch.from_numpy(S.values).to(dev)
        if not on_gpu:  # gloo broadcasts in place on the source too: never alias the caller's arrays
            ro, va = ro.clone(), va.clone()
    else:
        meta = torch.zeros(3, dtype=torch.int64, device=dev)
    dist.broadcast(meta, src, group=group)
    n_rows, n_cols, nnz = (int(x) for x in meta.tolist())
    if rank != src:
        ro = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(nnz, dtype=torch.int32, device=dev)
        va = torch.empty(nnz, dtype=torch.float64, device=dev)
    for t in (ro, ci, va):
        dist.broadcast(t, src, group=group)
    if on_gpu:
        from .device_build import DeviceCSR

        return DeviceCSR(n_rows, n_cols, ro, ci, va)
    return SparseMatrix(n_rows, n_cols, ro.numpy(), ci.numpy().astype(np.int64), va.numpy(), check=False)


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
    dt = "float64" if dtype == "f64" else "float32"
    if hasattr(S, "to_device_matrix"):  # a DeviceCSR (e.g. from broadcast_matrix): upload device to device
        dm = S.to_device_matrix(dt, device)
    else:
        dm = DeviceMatrix(S, dt, device)
    plan = dm.plan(hi - lo)
    plan.run(coeffs, n_stages, omega_kind=_OMEGA[omega_kind], seed=seed, col0=lo, d_global=d)
    peaks, _, _ = plan.diagnostics()
    tdt = torch.float64 if dtype == "f64" else torch.float32
    # every torch / NCCL op below runs on the library stream, so the gather, the
    # concatenation and K4 are ordered after the recurrence on the device (the
    # library stream is non-blocking: nothing orders it with torch's own stream)
    with torch.cuda.stream(dm.ctx.torch_stream()):
        local = torch.empty((S.n_rows, hi - lo), dtype=tdt, device=f"cuda:{device}")
        plan.copy_output_to(local.data_ptr(), hi - lo)
        E = assemble_columns(local, world, d, dtype, group)
        if normalize_rows:
            _lib.check(dm.lib.csemb_rownorm(dm.ctx.handle, E.data_ptr(), E.shape[0], d, d,
                                            _lib.F64 if dtype == "f64" else _lib.F32), "csemb_rownorm")
    dm.ctx.sync()
    dm.close()
    return E, combine_peaks(peaks, group)


# ---------------------------------------------------------------------------
# Row partition (config 5: graphs larger than one GPU's HBM)
# ---------------------------------------------------------------------------
def row_blocks(n: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Contiguous row blocks of n_pad = ceil(n / world) rows (the last may be
    shorter): the layout NCCL's equal-chunk all-gather needs."""
    if n < 1 or world < 1:
        raise ValueError("n and world must be positive")
    n_pad = -(-n // world)
    return n_pad, [(min(p * n_pad, n), min((p + 1) * n_pad, n)) for p in range(world)]


def local_rows(S, lo: int, hi: int):
    """Rows [lo, hi) of a CSR with their GLOBAL column ids (a rank's block)."""
    from .sparse import SparseMatrix

    S = SparseMatrix.of(S)
    offs = S.row_offsets[lo:hi + 1]
    return SparseMatrix(hi - lo, S.n_cols, offs - offs[0], S.col_indices[offs[0]:offs[-1]],
                        S.values[offs[0]:offs[-1]], check=False)


class DeviceRowEngine:
    """One rank's share of a row-partitioned run on its GPU (C ABI step-wise
    plan over caller-owned torch buffers)."""

    def __init__(self, S_local, row0, n_global, d, dtype, device, F, q, peers=None, mc=None, defer=False):
        from .engine import DeviceMatrix

        self.dm = DeviceMatrix(S_local, "float64" if dtype == "f64" else "float32", device)
        self.plan = self.dm.plan(d)
        self.row0, self.n_global = row0, n_global
        if mc is not None:  # fused exchange through NVLS multicast addresses of F[0], F[1]
            self.plan.partition_multicast(row0, n_global, (F[0].data_ptr(), F[1].data_ptr()), mc)
        elif peers is not None:  # fused exchange: F = this rank's two full buffers, peers = (parity-0, parity-1) pointer lists
            self.plan.partition_peers(row0, n_global, (F[0].data_ptr(), F[1].data_ptr()), peers[0], peers[1])
        elif not defer:
            self.bind(F, q)
        self.n_local, self.d = S_local.n_rows, d

    def bind(self, F, q, split: bool = False):
        """All-gather exchange: steps gather from F and write the local Q(r) to
        q[r & 1]; split=True also cuts the row block at its own column range
        (step_local before the all-gather completes, step after it)."""
        if split:
            self.plan.partition_split(self.row0, self.n_global, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
        else:
            self.plan.partition(self.row0, self.n_global, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())

    def step_local(self, r):
        self.plan.step_local(r)

    def begin(self, coeffs, omega_kind, seed, col0, d_global):
        self.plan.begin(coeffs, omega_kind=omega_kind, seed=seed, col0=col0, d_global=d_global)

    def step(self, r):
        # enqueued on the library stream; the caller's exchange is ordered after
        # it on the device (the driver runs its collectives on this stream)
        self.plan.step(r)

    def stream(self):
        return self.dm.ctx.torch_stream()

    def end(self, normalize_rows):
        import torch

        self.plan.end(normalize_rows)
        out = torch.empty((self.n_local, self.d), dtype=torch.float64 if self.dm.dtype == 0 else torch.float32,
                          device=f"cuda:{self.dm.ctx.device}")
        self.plan.copy_output_to(out.data_ptr(), self.d)
        self.dm.ctx.sync()
        peaks, _, _ = self.plan.diagnostics()
        self.dm.close()
        return out, peaks


def peer_buffers(shape, dtype, device, group, multicast: bool = False):
    """Two replicated full buffers in torch symmetric memory (NVLink-mapped on
    every rank) and, per parity, the device pointers of the peers' copies --
    or, with multicast=True, the NVLS multicast address of each buffer."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    group = dist.group.WORLD if group is None else group
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    F, peers, mc = [], ([], []), []
    for parity in range(2):
        t = symm_mem.empty(*shape, dtype=dtype, device=device)
        t.zero_()
        hdl = symm_mem.rendezvous(t, group)
        F.append(t)
        if multicast:
            base = int(hdl.multicast_ptr or 0)  # 0: no multicast object (no NVSwitch / driver support)
            if not base:
                raise RuntimeError("NVLS multicast is not available for this group")
            mc.append(base + (t.data_ptr() - hdl.buffer_ptrs[rank]))
        for p in range(world):
            if p != rank:
                peers[parity].append(hdl.get_buffer(p, list(shape), dtype).data_ptr())
    return F, (mc if multicast else peers)


def embed_row_partitioned(S_local, row0: int, n_global: int, coeffs, d: int, *, seed: int = 0,
                          omega_kind: str = "reference", dtype: str = "f64", normalize_rows: bool = False,
                          group=None, device: int | None = None, engine_factory=None, exchange: str = "allgather",
                          col0: int = 0, d_global: int | None = None):
    """E rows [row0, row0 + n_local) of f_L(S) Omega for a row-partitioned S.

    Each rank holds its row block of S (global column ids); every step gathers
    from a replicated full Q(r-1) that one all-gather of the ranks' local Q(r)
    refreshes -- the one exchange per step.  The
    projection is generated from the global row index on every rank, so no
    exchange precedes step 1.  Per-row arithmetic is unchanged, so the
    assembled E is bit-identical to the single-GPU result.  Returns the local
    E rows (torch tensor) and the per-chunk diagnostics max-combined over ranks.

    exchange="allgather": one NCCL all-gather of the local Q(r) per step.
    exchange="peer": the fused exchange -- K1's epilogue stores every Q(r) row
    into all ranks' replicated buffers over NVLink (torch symmetric memory),
    so the transfer overlaps the step; one barrier per step.  GPU only.
    exchange="multicast": the same through NVLS multicast (one multimem store
    per row, replicated by the NVSwitch).
    exchange="split": the all-gather overlapped with compute (SURVEY 8(e)
    "Overlap"): each rank's row block is cut at its own column range; the
    entries with local columns run from the rank's own Q(r-1) rows while the
    all-gather of Q(r-1) is in flight (on a separate stream), the remaining
    entries and the fused epilogue after it.  Local columns are summed first,
    so E agrees with one GPU within rounding (bit-identical to the split-order
    restatement), not bit for bit.
    col0 / d_global: the d columns are the slice [col0, col0 + d) of a
    d_global-column projection (the 2-D layout, `embed_2d`).
    """
    import torch
    import torch.distributed as dist

    from . import _lib

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n_pad, blocks = row_blocks(n_global, world)
    if blocks[rank] != (row0, row0 + S_local.n_rows):
        raise ValueError(f"rank {rank} must hold rows {blocks[rank]}, not [{row0}, {row0 + S_local.n_rows})")
    if omega_kind not in ("reference", "philox"):
        raise ValueError("the row-partitioned driver generates the projection (reference or philox)")
    width = 2 if dtype == "f64" else 4
    ld = -(-d // width) * width
    tdt = torch.float64 if dtype == "f64" else torch.float32
    on_gpu = engine_factory is None
    dev = torch.device(f"cuda:{torch.cuda.current_device() if device is None else device}") if on_gpu \
        else torch.device("cpu")
    if exchange not in ("allgather", "peer", "multicast", "split"):
        raise ValueError("exchange must be 'allgather', 'peer', 'multicast' or 'split'")
    if exchange in ("peer", "multicast"):
        if not on_gpu:
            raise ValueError("the fused peer exchange runs on GPUs (torch symmetric memory)")
        mcast = exchange == "multicast"
        F2, ptrs = peer_buffers((world * n_pad, ld), tdt, dev, group, multicast=mcast)
        torch.cuda.synchronize(dev)  # the buffers' zero-fill (torch's stream) before any library-stream write
        eng = DeviceRowEngine(S_local, row0, n_global, d, dtype, dev.index, F2, None,
                              peers=None if mcast else ptrs, mc=ptrs if mcast else None)
        kind = _lib.OMEGA_SPLITMIX if omega_kind == "reference" else _lib.OMEGA_PHILOX
        with torch.cuda.stream(eng.stream()):
            eng.begin(coeffs, kind, seed, col0, d if d_global is None else d_global)
            flag = torch.zeros(1, device=dev)
            for r in range(1, len(coeffs)):
                eng.step(r)
                if r < len(coeffs) - 1:
                    # device-side barrier: the all-reduce starts after this rank's step-r
                    # kernels (which end with a system-scope fence) and completes only
                    # when every rank has reached it; step r+1 waits for it on the
                    # stream.  No host synchronisation per step.
                    dist.all_reduce(flag, group=group)
            E, peaks = eng.end(normalize_rows)
        return E, combine_peaks(peaks, group)
    if on_gpu:
        eng = DeviceRowEngine(S_local, row0, n_global, d, dtype, dev.index, None, None, defer=True)
        stream = eng.stream()
    else:
        stream = None
    order = len(coeffs) - 1
    kind = _lib.OMEGA_SPLITMIX if omega_kind == "reference" else _lib.OMEGA_PHILOX
    # On GPUs the buffers, the steps and the per-step all-gather all run on the
    # library stream: the all-gather of Q(r) starts when step r's kernels finish
    # and step r+1 starts when it completes, ordered on the device with no host
    # synchronisation in the loop.
    split = exchange == "split"
    with (torch.cuda.stream(stream) if stream is not None else _nullcontext()):
        F = torch.zeros((world * n_pad, ld), dtype=tdt, device=dev)
        q = [torch.zeros((n_pad, ld), dtype=tdt, device=dev) for _ in range(2)]
        if on_gpu:
            eng.bind(F, q, split=split)
        else:
            eng = engine_factory(S_local, row0, n_global, d, dtype, F, q)
        eng.begin(coeffs, kind, seed, col0, d if d_global is None else d_global)
        parts = [F[p * n_pad:(p + 1) * n_pad] for p in range(world)]
        nccl = dist.get_backend(group) == "nccl"
        # split: the all-gather runs on its own stream, after the step that wrote
        # Q(r); the library stream meanwhile runs step r+1's local-column part and
        # waits for the all-gather only before the remote part
        comm = torch.cuda.Stream(device=dev) if (split and on_gpu) else None

        def gather(r):
            if comm is not None:
                comm.wait_stream(stream)  # Q(r) is written
                with torch.cuda.stream(comm):
                    dist.all_gather_into_tensor(F, q[r & 1], group=group)
            elif nccl:
                dist.all_gather_into_tensor(F, q[r & 1], group=group)
            else:
                dist.all_gather(parts, q[r & 1], group=group)

        for r in range(1, order + 1):
            if split:
                eng.step_local(r)  # this rank's own Q(r-1) rows: no exchange needed
                if comm is not None:
                    stream.wait_stream(comm)  # the all-gather of Q(r-1) has landed in F
            eng.step(r)
            if r < order:  # refresh the replicated Q(r) for the next step
                gather(r)
        E, peaks = eng.end(normalize_rows)
    return E, combine_peaks(peaks, group)


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


# ---------------------------------------------------------------------------
# 2-D layout: row blocks x column shards
# ---------------------------------------------------------------------------
def grid_groups(R: int, C: int):
    """Sub-groups of an R x C rank grid (rank = rr * C + cc): for every column
    shard cc the R ranks that exchange Q(r) each step, for every row block rr
    the C ranks that assemble its columns at the end.  Collective: every rank
    creates every group, in the same order."""
    import torch.distributed as dist

    if R * C != dist.get_world_size():
        raise ValueError(f"grid {R} x {C} does not match world size {dist.get_world_size()}")
    row_groups = [dist.new_group([rr * C + cc for rr in range(R)]) for cc in range(C)]
    col_groups = [dist.new_group([rr * C + cc for cc in range(C)]) for rr in range(R)]
    return row_groups, col_groups


def embed_2d(S, coeffs, d: int, grid: tuple[int, int], *, seed: int = 0, omega_kind: str = "reference",
             dtype: str = "f64", normalize_rows: bool = True, device: int | None = None, engine_factory=None,
             exchange: str = "allgather", groups=None):
    """E rows of this rank's row block (all d columns) on an R x C rank grid.

    Column sharding replicates the whole matrix and leaves every rank the full
    per-row work on d/N columns; the row partition exchanges all of Q(r) every
    step.  The grid trades the two: rank (rr, cc) holds row block rr of S
    (global column ids) and runs the row-partitioned recurrence on column
    shard cc with the R ranks of its shard (one exchange of Q(r) per step, R x
    smaller than the 1-D row partition's), then the C ranks of its row block
    all-gather their column slices and K4 normalises the assembled rows.
    Every element is computed exactly as on one GPU: bit-identical results.
    `groups` = grid_groups(R, C) (create them once and reuse)."""
    import torch
    import torch.distributed as dist

    R, C = grid
    rank = dist.get_rank()
    rr, cc = divmod(rank, C)
    row_groups, col_groups = groups if groups is not None else grid_groups(R, C)
    _, blocks = row_blocks(S.n_rows, R)
    lo_r, hi_r = blocks[rr]
    align = 2 if dtype == "f64" else 4
    lo_c, hi_c = column_shards(d, C, align)[cc]
    S_local = local_rows(S, lo_r, hi_r)
    E_local, peaks = embed_row_partitioned(
        S_local, lo_r, S.n_rows, coeffs, hi_c - lo_c, seed=seed, omega_kind=omega_kind, dtype=dtype,
        normalize_rows=False, group=row_groups[cc], device=device, engine_factory=engine_factory,
        exchange=exchange, col0=lo_c, d_global=d)
    E = assemble_columns(E_local, C, d, dtype, group=col_groups[rr])
    if normalize_rows and E.shape[0] > 0:
        if E.is_cuda:
            from . import _lib

            ctx = _lib.context(E.device.index)
            torch.cuda.synchronize(E.device)
            _lib.check(ctx.lib.csemb_rownorm(ctx.handle, E.data_ptr(), E.shape[0], d, d,
                                             _lib.F64 if dtype == "f64" else _lib.F32), "csemb_rownorm")
            ctx.sync()
        else:  # CPU tests (oracle engine): the reference cosine harness's normalisation
            nrm = torch.linalg.norm(E, dim=1, keepdim=True)
            E = torch.where(nrm > 0, E / torch.where(nrm > 0, nrm, torch.ones_like(nrm)), torch.zeros_like(E))
    return E, combine_peaks(peaks, col_groups[rr])

