"""K1 against its same-data gather floor (csemb_diag_gather_csr) at
config-2 size, per graph / dtype / width:

    python tools/probe_floor.py [--dtype f64,f32] [--graphs sbm,random,band] [--widths 80]

floor = the time to fetch, for every stored entry in stored order, the whole
gathered row with no arithmetic / epilogue / streams (4 or 8 entries in
flight per lane group).
"""

import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64,f32")
ap.add_argument("--L", type=int, default=12)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--graphs", default="sbm,random,band")
ap.add_argument("--widths", default="80")
args = ap.parse_args()
n = args.n


def ring(n, w):
    base = np.arange(n, dtype=np.int64)
    return np.concatenate([np.stack([base, (base + k) % n], 1) for k in range(1, w + 1)])


makers = {
    "band": lambda: pb.normalized_adjacency(ring(n, 10), n),
    "sbm": lambda: graphs.sbm(n, 100, 15.0, 5.0, seed=2),
    "random": lambda: pb.normalized_adjacency(np.random.default_rng(1).integers(0, n, size=(10 * n, 2)), n),
}
coeffs = pb.legendre_coefficients(pb.indicator_above(0.95), args.L).coeffs
for name in args.graphs.split(","):
    S = makers[name]()
    for dt, w in [(dt, int(w)) for dt in args.dtype.split(",") for w in args.widths.split(",")]:
        dm = pb.DeviceMatrix(S, "float64" if dt == "f64" else "float32")
        plan = dm.plan(w)
        best = 1e9
        for _ in range(3):
            plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7)
            dm.ctx.sync()
            tot, steps, launches = plan.timing()
            best = min(best, steps / (len(coeffs) - 1))
        es = 8 if dt == "f64" else 4
        W = 16 // es
        row_bytes = (w + W - 1) // W * W * es
        fl = {}
        for depth in (4, 8):
            ms, gbs = C.c_double(), C.c_double()
            _lib.check(dm.lib.csemb_diag_gather_csr(dm.handle, row_bytes, depth, C.byref(ms), C.byref(gbs)), "floor")
            fl[depth] = (ms.value, gbs.value)
        fmin = min(v[0] for v in fl.values())
        print(f"{name:7s} {dt} d={w}: nnz {S.nnz}  K1 {best:.4f} ms/step | gather floor "
              + "  ".join(f"U={k}: {v[0]:.4f} ms ({v[1]:.0f} GB/s)" for k, v in fl.items())
              + f" | K1/floor {best / fmin:.3f}", flush=True)
        dm.close()
