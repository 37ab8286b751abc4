"""Short config-3 / config-4 run for ncu: a few fused K1 steps at full scale.

    python tools/profile_cfg.py --config 4 --dtype f32 --L 3
    ncu --set full -k regex:"k_step|k_heavy" -c 3 -o prof python tools/profile_cfg.py ...

The inputs are built on the device exactly as tools/bench_configs.py builds
them; config 4 is scaled by the 30-iteration norm estimate recorded in
profiles/r1_configs34.json instead of re-running it (the profile is of K1).
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, device_build as db  # noqa: E402
from bench_configs import CutAbove  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--L", type=int, default=3)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--split", default=None, help="comma list of split thresholds to run in turn (0 = never split)")
args = ap.parse_args()

if args.config == 3:
    S = db.normalized_adjacency(db.chung_lu_edges(10_000_000, seed=3), 10_000_000)
    f, d, scale = pb.commute_time(0.01), 80, 1.0
else:
    S = db.dilate(db.bag_of_words(2_000_000, 500_000, seed=4))
    f, d, scale = pb.odd_extension(CutAbove(0.3)), 96, 1.0 / 130.35983614177252
torch.cuda.synchronize()
dm = S.to_device_matrix("float64" if args.dtype == "f64" else "float32")
if scale != 1.0:
    dm.scale(scale)
coeffs = pb.legendre_coefficients(f, args.L).coeffs
plan = dm.plan(d)
for thr in ([None] if args.split is None else [int(x) for x in args.split.split(",")]):
    if thr is not None:
        plan.set_load_balance(split_threshold=thr)
    for _ in range(args.reps):
        plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7)
        dm.ctx.sync()
        tot, steps, launches = plan.timing()
        print(f"config {args.config} {args.dtype} split={thr}: K1 {steps / args.L:.3f} ms/step "
              f"({launches // args.L} launches/step)", flush=True)
dm.close()
