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
