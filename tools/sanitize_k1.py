"""Small K1 workloads covering every schedule path, for compute-sanitizer.

    python tools/sanitize_k1.py && compute-sanitizer --tool memcheck python tools/sanitize_k1.py

Covers: bucketed row permutation with the reverse sweep, split heavy rows
(chunk pass + combine), warps whose rows are all empty, column tiles, both
dtypes, exact peaks, and the norm estimate's SpMM.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import graphs  # noqa: E402

rng = np.random.default_rng(0)
n = 30011  # not a multiple of any rows-per-warp
e = np.concatenate([graphs.chung_lu_edges(n, seed=1),
                    np.stack([np.full(6000, 7, np.int64), rng.integers(0, n, 6000)], 1)])
S = pb.normalized_adjacency(e, n)
print("nnz", S.nnz, "max row", int(np.diff(S.row_offsets).max()), "empty rows", int((np.diff(S.row_offsets) == 0).sum()))
th = pb.legendre_coefficients(pb.commute_time(0.01), 7).coeffs
for dt in ("float64", "float32"):
    dm = pb.DeviceMatrix(S, dt)
    for d in (24, 80, 200):
        om = pb.sample_projection(n, d, 3)
        plan = dm.plan(d)
        for thr, order, exact in ((4096, -1, False), (64, 1, True), (0, 0, False)):
            plan.set_load_balance(thr, order)
            plan.set_exact_peaks(exact)
            out = plan.apply(th, 2, om, normalize_rows=True)
            assert np.all(np.isfinite(out))
    print(dt, "norm", dm.spectral_norm(5, 20, 1))
    dm.close()
print("ok")

# round 2: the split exchange (device column split + split combine), the
# value-free check and the same-data gather floor
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_1509_08360_b200 import _lib  # noqa: E402
from paper_1509_08360_b200.distributed import local_rows, row_blocks  # noqa: E402

for dt, tdt in (("float64", torch.float64), ("float32", torch.float32)):
    world, d = 3, 40
    n_pad, blocks = row_blocks(n, world)
    F = torch.zeros((world * n_pad, d), dtype=tdt, device="cuda")
    for lo, hi in blocks:
        dm = pb.DeviceMatrix(local_rows(S, lo, hi), dt)
        plan = dm.plan(d)
        q = [torch.zeros((n_pad, d), dtype=tdt, device="cuda") for _ in range(2)]
        plan.partition_split(lo, n, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
        torch.cuda.synchronize()
        plan.begin(th, omega_kind=1, seed=3)
        for r in range(1, len(th)):
            plan.step_local(r)
            plan.step(r)
        plan.end(True)
        assert np.all(np.isfinite(plan.download()))
        dm.close()
    dm = pb.DeviceMatrix(S, dt)
    print(dt, "value_free", dm.value_free)
    for depth in (4, 8):
        ms, gbs = C.c_double(), C.c_double()
        _lib.check(dm.lib.csemb_diag_gather_csr(dm.handle, 80 * (8 if dt == "float64" else 4), depth,
                                                C.byref(ms), C.byref(gbs)), "floor")
    dm.close()
print("ok (round 2 paths)")
