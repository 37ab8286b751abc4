"""Short config-2 run for ncu: a few fused K1 steps on the bench workload.

    python tools/profile_k1.py --dtype f64 --L 6
    ncu --set full -k regex:k_step -s 3 -c 1 -o prof python tools/profile_k1.py ...
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64")
ap.add_argument("--L", type=int, default=6)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=80)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()

S = graphs.sbm(args.n, 100, 15.0, 5.0, seed=2)
coeffs = pb.legendre_coefficients(pb.indicator_above(0.95), args.L).coeffs
dm = pb.DeviceMatrix(S, "float64" if args.dtype == "f64" else "float32")
plan = dm.plan(args.d)
for _ in range(args.reps):
    t0 = time.perf_counter()
    plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7, normalize_rows=True)
    dm.ctx.sync()
    tot, steps, launches = plan.timing()
    print(f"{args.dtype}: L={args.L} total {tot:.3f} ms, K1 avg {steps / max(launches, 1):.3f} ms "
          f"({launches} launches), wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)

if os.environ.get("CSEMB_PROFILE_FLOOR"):  # the same-data gather floor (csemb_diag_gather_csr), for ncu
    import ctypes as C

    es = 8 if args.dtype == "f64" else 4
    W = 16 // es
    ms, gbs = C.c_double(), C.c_double()
    _lib.check(dm.lib.csemb_diag_gather_csr(dm.handle, (args.d + W - 1) // W * W * es, 4, C.byref(ms), C.byref(gbs)),
               "floor")
    print(f"gather floor {ms.value:.4f} ms ({gbs.value:.0f} GB/s)")
