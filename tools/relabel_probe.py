"""Does a degree-ordered vertex relabel help K1 on config 3?

    python tools/relabel_probe.py [--dtype f32,f64] [--L 20]

Relabels the config-3 Chung-Lu graph so vertices are numbered by descending
degree, keeping every row's stored entry order (columns are mapped, not
re-sorted, so the per-row summation order -- and the result, up to the row
permutation -- is unchanged), and times K1 per step on both labelings.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, device_build as db  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f32,f64")
ap.add_argument("--L", type=int, default=20)
ap.add_argument("--n", type=int, default=10_000_000)
args = ap.parse_args()

n = args.n
H = db.normalized_adjacency(db.chung_lu_edges(n, seed=3), n).to_host()
torch.cuda.empty_cache()
ro, ci, va = H.row_offsets, H.col_indices, H.values
lens = np.diff(ro)
inv = np.argsort(-lens, kind="stable")          # new id p -> old vertex inv[p]
rank = np.empty(n, dtype=np.int64)
rank[inv] = np.arange(n)
new_lens = lens[inv]
new_ro = np.zeros(n + 1, dtype=np.int64)
np.cumsum(new_lens, out=new_ro[1:])
# entry order: old rows in new order, each row's entries in stored order
starts = np.repeat(ro[inv] - new_ro[:-1], new_lens)
idx = np.arange(len(va), dtype=np.int64) + starts
new_ci = rank[ci[idx]]
new_va = va[idx]
th = pb.legendre_coefficients(pb.commute_time(0.01), args.L).coeffs
for dt in args.dtype.split(","):
    res = {}
    for name, (r, c, v) in (("original", (ro, ci, va)), ("degree-ordered", (new_ro, new_ci, new_va))):
        S = pb.SparseMatrix(n, n, r, c, v, check=False)
        dm = pb.DeviceMatrix(S, "float64" if dt == "f64" else "float32")
        plan = dm.plan(80)
        best = 1e9
        for _ in range(3):
            plan.run(th, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7)
            dm.ctx.sync()
            best = min(best, plan.timing()[1] / args.L)
        res[name] = best
        if name == "original":
            E0 = plan.download()
        else:
            E1 = plan.download()
        dm.close()
    # Philox Omega hashes the (new) row index, so compare only the timing here
    print(f"config 3 {dt}: K1 per step original {res['original']:.3f} ms, degree-ordered "
          f"{res['degree-ordered']:.3f} ms ({res['degree-ordered'] / res['original']:.3f}x)", flush=True)
