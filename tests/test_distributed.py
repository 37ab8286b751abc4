"""Column-sharded multi-rank path on CPU (gloo, world_size 2).

The per-rank compute is injected (the oracle stands in for the GPU kernel, as
allowed for tests); what is under test is the host-side distributed logic of
paper_1509_08360_b200.distributed: shard boundaries, global-d hashing of each
rank's projection slice, the all-gather assembly, and the max-combination of
per-chunk diagnostics.  The assembled E must equal the single-process result
bit-for-bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1509_08360_b200.distributed import column_shards


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(3)
    n = 300
    dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.05)
    dense = 0.5 * (dense + dense.T)
    dense /= np.abs(np.linalg.eigvalsh(dense)).max() * 1.05
    import scipy.sparse as sp

    csr = sp.csr_array(dense)
    csr.sort_indices()
    S = O.CSR(n, n, csr.indptr, csr.indices, csr.data)
    coeffs = np.random.default_rng(4).standard_normal(13) * 0.3
    return S, coeffs


def _local_compute(S, coeffs, d, seed, lo, hi, dtype):
    """Oracle stand-in for one rank: columns [lo, hi) hashed with the global d,
    plus per-GLOBAL-chunk peaks (columns are independent, so each chunk slice
    is run on its own)."""
    order = len(coeffs) - 1
    n_chunks = (d + 31) // 32
    block = O.sample_projection(S.n_rows, d, seed, col0=lo, w=hi - lo)
    E, _, _ = O.run_stage(S, coeffs, block)
    peaks = np.zeros((1, order, n_chunks))
    for ch in range(lo // 32, (hi - 1) // 32 + 1):
        a, b = max(lo, 32 * ch), min(hi, 32 * ch + 32)
        _, pk, _ = O.run_stage(S, coeffs, block[:, a - lo:b - lo])
        peaks[0, :, ch] = pk[:, 0]
    tdt = torch.float64 if dtype == "f64" else torch.float32
    return torch.from_numpy(E).to(tdt), peaks


def _worker(rank, world, port, d, seed, dtype, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import embed_column_sharded

        S, coeffs = _problem()
        E, peaks = embed_column_sharded(
            S, coeffs, d, seed=seed, dtype=dtype, normalize_rows=False,
            compute=lambda lo, hi: _local_compute(S, coeffs, d, seed, lo, hi, dtype))
        if rank == 0:
            np.savez(result_path, E=E.numpy().astype(np.float64), peaks=peaks)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,dtype", [(70, "f64"), (80, "f32"), (5, "f64")])
def test_column_sharded_matches_single_process(tmp_path, d, dtype):
    world, seed = 2, 11
    out = str(tmp_path / "r.npz")
    mp.start_processes(_worker, args=(world, _free_port(), d, seed, dtype, out), nprocs=world,
                       start_method="spawn", join=True)
    got = np.load(out)
    S, coeffs = _problem()
    ref, ref_peaks, _ = O.run_stage(S, coeffs, O.sample_projection(S.n_rows, d, seed))
    if dtype == "f64":
        assert np.array_equal(got["E"], ref)
    else:
        assert np.array_equal(got["E"], ref.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(got["peaks"][0], ref_peaks)


def test_shard_boundaries():
    for d in (1, 5, 40, 70, 80, 96, 517):
        for world in (1, 2, 3, 4, 8):
            for align in (1, 2, 4):
                sh = column_shards(d, world, align)
                assert sh[0][0] == 0 and sh[-1][1] == d and len(sh) == world
                assert all(a <= b for a, b in sh)
                assert all(sh[i][1] == sh[i + 1][0] for i in range(world - 1))
                assert all(lo % align == 0 for lo, _ in sh)
    assert column_shards(80, 8, 2) == [(i * 10, i * 10 + 10) for i in range(8)]
    with pytest.raises(ValueError):
        column_shards(0, 2, 2)


# ---------------------------------------------------------------------------
# row partition (config 5 layout), oracle engine on CPU
# ---------------------------------------------------------------------------
class OracleRowEngine:
    """CPU stand-in for DeviceRowEngine: same buffers, oracle arithmetic
    (numpy restatement of one engine._run_stage step)."""

    def __init__(self, S_local, row0, n_global, d, dtype, F, q):
        self.S = O.CSR.of(S_local)
        self.row0, self.n, self.N, self.d, self.F, self.q = row0, S_local.n_rows, n_global, d, F, q

    def begin(self, coeffs, kind, seed, col0, d_global):
        assert kind == 1  # reference hash
        self.coeffs = coeffs
        full = O.sample_projection(self.N, d_global, seed, col0, self.d)  # columns [col0, col0 + d)
        self.F[:self.N, :self.d] = torch.from_numpy(full)
        q0 = full[self.row0:self.row0 + self.n]
        self.q[0][:self.n, :self.d] = torch.from_numpy(q0)
        self.E = coeffs[0] * q0
        self.peaks = np.zeros((1, len(coeffs) - 1, (d_global + 31) // 32))

    def step(self, r):
        y = O.spmm(self.S, np.ascontiguousarray(self.F[:self.N, :self.d].numpy()))
        alpha, beta = 2.0 - 1.0 / r, 1.0 - 1.0 / r
        q = alpha * y
        if r > 1:
            q = q - beta * self.q[r & 1][:self.n, :self.d].numpy()
        self.E = self.E + self.coeffs[r] * q
        self.q[r & 1][:self.n, :self.d] = torch.from_numpy(q)

    def end(self, normalize_rows):
        return torch.from_numpy(self.E), self.peaks


class OracleSplitRowEngine(OracleRowEngine):
    """CPU stand-in for the split exchange (csemb_plan_partition_split):
    step_local sums the local-column entries from this rank's own Q(r-1) rows,
    step adds the remote-column sums from the refreshed full buffer."""

    def __init__(self, S_local, row0, n_global, d, dtype, F, q):
        from conftest import split_csr

        super().__init__(S_local, row0, n_global, d, dtype, F, q)
        self.Sl, self.Sr = split_csr(self.S, row0, row0 + self.n, rows=(0, self.n))
        self.yl = None

    def step_local(self, r):
        self.yl = O.spmm(self.Sl, np.ascontiguousarray(self.q[(r - 1) & 1][:self.n, :self.d].numpy()))

    def step(self, r):
        y = self.yl + O.spmm(self.Sr, np.ascontiguousarray(self.F[:self.N, :self.d].numpy()))
        self.yl = None
        q = (2.0 - 1.0 / r) * y
        if r > 1:
            q = q - (1.0 - 1.0 / r) * self.q[r & 1][:self.n, :self.d].numpy()
        self.E = self.E + self.coeffs[r] * q
        self.q[r & 1][:self.n, :self.d] = torch.from_numpy(q)


def _split_worker(rank, world, port, d, seed, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import embed_row_partitioned, local_rows, row_blocks

        S, coeffs = _problem()
        _, blocks = row_blocks(S.n_rows, world)
        lo, hi = blocks[rank]
        Sl = local_rows(_as_sparse(S), lo, hi)
        E, _ = embed_row_partitioned(Sl, lo, S.n_rows, coeffs, d, seed=seed, engine_factory=OracleSplitRowEngine,
                                     exchange="split")
        np.save(result_path + f".{rank}.npy", E.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_exchange_matches_split_order_and_single_process(tmp_path, world):
    # the overlapped exchange (local columns first, SURVEY 8(e) "Overlap"):
    # bit-identical to the split-order restatement, within rounding of the
    # single-process stored order
    from conftest import split_order_stage
    from paper_1509_08360_b200.distributed import row_blocks

    d, seed = 37, 5
    out = str(tmp_path / "split")
    mp.start_processes(_split_worker, args=(world, _free_port(), d, seed, out), nprocs=world,
                       start_method="spawn", join=True)
    got = np.concatenate([np.load(out + f".{p}.npy") for p in range(world)])
    S, coeffs = _problem()
    om = O.sample_projection(S.n_rows, d, seed)
    _, blocks = row_blocks(S.n_rows, world)
    assert np.array_equal(got, split_order_stage(S, coeffs, om, blocks))
    ref, _, _ = O.run_stage(S, coeffs, om)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def _row_worker(rank, world, port, d, seed, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import embed_row_partitioned, local_rows, row_blocks

        S, coeffs = _problem()
        _, blocks = row_blocks(S.n_rows, world)
        lo, hi = blocks[rank]
        Sl = local_rows(_as_sparse(S), lo, hi)
        E, _ = embed_row_partitioned(Sl, lo, S.n_rows, coeffs, d, seed=seed, engine_factory=OracleRowEngine)
        np.save(result_path + f".{rank}.npy", E.numpy())
    finally:
        dist.destroy_process_group()


def _as_sparse(S):
    from paper_1509_08360_b200 import SparseMatrix

    return SparseMatrix(S.n_rows, S.n_cols, S.row_offsets, S.col_indices, S.values)


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_matches_single_process(tmp_path, world):
    d, seed = 37, 5
    out = str(tmp_path / "rows")
    mp.start_processes(_row_worker, args=(world, _free_port(), d, seed, out), nprocs=world,
                       start_method="spawn", join=True)
    got = np.concatenate([np.load(out + f".{p}.npy") for p in range(world)])
    S, coeffs = _problem()
    ref, _, _ = O.run_stage(S, coeffs, O.sample_projection(S.n_rows, d, seed))
    assert np.array_equal(got, ref)


def test_row_blocks():
    from paper_1509_08360_b200.distributed import row_blocks

    assert row_blocks(10, 3) == (4, [(0, 4), (4, 8), (8, 10)])
    assert row_blocks(2, 4) == (1, [(0, 1), (1, 2), (2, 2), (2, 2)])


def _exchange_arg_worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import embed_row_partitioned, local_rows, row_blocks

        S, coeffs = _problem()
        _, blocks = row_blocks(S.n_rows, world)
        lo, hi = blocks[rank]
        Sl = local_rows(_as_sparse(S), lo, hi)
        msgs = []
        for exchange in ("peer", "ring"):  # peer: GPUs only (symmetric memory); ring: unknown
            try:
                embed_row_partitioned(Sl, lo, S.n_rows, coeffs, 8, engine_factory=OracleRowEngine, exchange=exchange)
                msgs.append("no error")
            except ValueError as e:
                msgs.append(str(e))
        with open(result_path + f".{rank}.txt", "w") as fh:
            fh.write("\n".join(msgs))
    finally:
        dist.destroy_process_group()


def test_row_partitioned_exchange_argument(tmp_path):
    out = str(tmp_path / "ex")
    mp.start_processes(_exchange_arg_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    for p in range(2):
        msgs = open(out + f".{p}.txt").read().split("\n")
        assert "GPUs" in msgs[0] and "exchange must be" in msgs[1]


# ---------------------------------------------------------------------------
# 2-D layout (row blocks x column shards), oracle engine on CPU
# ---------------------------------------------------------------------------
def _grid_worker(rank, world, port, grid, d, seed, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import embed_2d, grid_groups

        S, coeffs = _problem()
        groups = grid_groups(*grid)
        E, peaks = embed_2d(_as_sparse(S), coeffs, d, grid, seed=seed, engine_factory=OracleRowEngine,
                            normalize_rows=False, groups=groups)
        np.save(result_path + f".{rank}.npy", E.numpy())
        En, _ = embed_2d(_as_sparse(S), coeffs, d, grid, seed=seed, engine_factory=OracleRowEngine, groups=groups)
        np.save(result_path + f".{rank}.norm.npy", En.numpy())
        # the split (overlapped) exchange through the grid driver
        Es, _ = embed_2d(_as_sparse(S), coeffs, d, grid, seed=seed, engine_factory=OracleSplitRowEngine,
                         normalize_rows=False, groups=groups, exchange="split")
        np.save(result_path + f".{rank}.split.npy", Es.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(2, 2), (1, 2), (2, 1)])
def test_2d_grid_matches_single_process(tmp_path, grid):
    from paper_1509_08360_b200.distributed import row_blocks

    d, seed = 37, 5
    world = grid[0] * grid[1]
    out = str(tmp_path / "grid")
    mp.start_processes(_grid_worker, args=(world, _free_port(), grid, d, seed, out), nprocs=world,
                       start_method="spawn", join=True)
    S, coeffs = _problem()
    ref, _, _ = O.run_stage(S, coeffs, O.sample_projection(S.n_rows, d, seed))
    _, blocks = row_blocks(S.n_rows, grid[0])
    for rank in range(world):
        lo, hi = blocks[rank // grid[1]]
        assert np.array_equal(np.load(out + f".{rank}.npy"), ref[lo:hi])  # every rank: its rows, all columns
        np.testing.assert_allclose(np.load(out + f".{rank}.norm.npy"), O.row_normalize(ref)[lo:hi], rtol=0,
                                   atol=1e-15)
    from conftest import split_order_stage

    split_ref = split_order_stage(S, coeffs, O.sample_projection(S.n_rows, d, seed), blocks)
    for rank in range(world):
        lo, hi = blocks[rank // grid[1]]
        assert np.array_equal(np.load(out + f".{rank}.split.npy"), split_ref[lo:hi])


def test_grid_shape_must_match_world(tmp_path):
    out = str(tmp_path / "bad")

    mp.start_processes(_bad_grid_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    for p in range(2):
        assert "does not match world size" in open(out + f".{p}.txt").read()


def _bad_grid_worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import grid_groups

        try:
            grid_groups(2, 2)
            msg = "no error"
        except ValueError as e:
            msg = str(e)
        with open(result_path + f".{rank}.txt", "w") as fh:
            fh.write(msg)
    finally:
        dist.destroy_process_group()



# ---------------------------------------------------------------------------
# C1: the matrix broadcast from one rank, then the column-sharded run
# ---------------------------------------------------------------------------
def _bcast_worker(rank, world, port, d, seed, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08360_b200.distributed import broadcast_matrix, embed_column_sharded

        S0, coeffs = _problem()
        S = broadcast_matrix(_as_sparse(S0) if rank == 1 else None, src=1)
        assert np.array_equal(S.row_offsets, S0.row_offsets)
        assert np.array_equal(S.col_indices, S0.col_indices) and S.col_indices.dtype == np.int64
        assert S.values.tobytes() == S0.values.tobytes()
        Sc = O.CSR.of(S)
        E, _ = embed_column_sharded(S, coeffs, d, seed=seed, normalize_rows=False,
                                    compute=lambda lo, hi: _local_compute(Sc, coeffs, d, seed, lo, hi, "f64"))
        np.save(result_path + f".{rank}.npy", E.numpy())
    finally:
        dist.destroy_process_group()


def test_broadcast_matrix_then_column_shards(tmp_path):
    d, seed, world = 21, 3, 3
    out = str(tmp_path / "bc")
    mp.start_processes(_bcast_worker, args=(world, _free_port(), d, seed, out), nprocs=world,
                       start_method="spawn", join=True)
    S, coeffs = _problem()
    ref, _, _ = O.run_stage(S, coeffs, O.sample_projection(S.n_rows, d, seed))
    for p in range(world):
        assert np.array_equal(np.load(out + f".{p}.npy"), ref)
