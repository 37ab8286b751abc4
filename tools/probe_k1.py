"""K1 time vs graph locality at config-2 size (n=1e6, ~20 nnz/row, d=80).

    python tools/probe_k1.py [--dtype f64] [--L 6]

band   : ring graph, neighbours i+-1..10 (every gather L2-resident)
sbm    : config 2 (75% intra-block, 25% uniform inter-block)
random : ~20 uniform random neighbours per row
"""

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64")
ap.add_argument("--L", type=int, default=6)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--graphs", default="band,sbm,random")
ap.add_argument("--widths", default="80")
ap.add_argument("--efold", type=int, default=None)
ap.add_argument("--reverse", type=int, default=None)
ap.add_argument("--row-order", type=int, default=None, help="-1 auto, 0 natural, 1 bucketed by batch count")
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
        if args.efold:
            plan.set_option(_lib.OPT_E_FOLD, args.efold)
        if args.reverse is not None:
            plan.set_option(_lib.OPT_REVERSE_SWEEP, args.reverse)
        if args.row_order is not None:
            plan.set_option(_lib.OPT_ROW_ORDER, args.row_order)
        best = 1e9
        for _ in range(3):
            plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7)
            dm.ctx.sync()
            tot, steps, launches = plan.timing()
            best = min(best, steps / launches)
        es = 8 if dt == "f64" else 4
        B = S.nnz * (4 + es) + 5 * n * w * es
        print(f"{name:7s} {dt} d={w}: nnz {S.nnz}  K1 {best:.3f} ms  (x{80 / w:.1f} panels = {best * 80 / w:.3f} ms "
              f"for 80 cols) -> {B / best / 1e6:.0f} GB/s algorithmic ({B / best / 1e6 / 6552:.2f} of 6552)", flush=True)
        dm.close()
