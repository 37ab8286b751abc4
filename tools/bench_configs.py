"""Full-scale configs 3 and 4 on one B200 (inputs built on the device).

    python tools/bench_configs.py [--configs 3,4] [--dtype f32] [--reps 2]

config 3: Chung-Lu n=1e7 (Pareto 2.1 degrees in [2, 1e4], mean 20),
          normalized adjacency, d=80, L=180, f = commute_time(clip=0.01).
config 4: bag-of-words 2e6 x 5e5 (Poisson(150) tokens, Zipf(1.1) terms,
          tf-idf, rows L2-normalised), dilation [0 A^T; A 0], spectral norm by
          30 power iterations on k = ceil(6 ln N) vectors, d=96, L=120,
          f(x) = x * 1{x >= 0.3} odd-extended.
Prints one JSON line per config with build/norm/embedding times, the K1 time
per recurrence step (all of its launches: heavy-row chunks, light rows,
heavy-row combine) and its fraction of the measured HBM roofline (algorithmic
bytes T*(4+val) + 5*N*d*dtype per step), plus the gather volume T*d*dtype that
actually crosses L2->SM each step.
"""

import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, device_build as db  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6552.0


class CutAbove:
    def __init__(self, c):
        self.c = c

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        return np.where(x >= self.c, x, 0.0)

    def breakpoints(self):
        return (self.c,)


ROW_ORDER = None


def run_embed(dm, coeffs, d, reps, dtype, normalize=True):
    plan = dm.plan(d)
    if ROW_ORDER is not None:
        plan.set_load_balance(row_order=ROW_ORDER)
    res = []
    for _ in range(reps + 1):
        plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7, normalize_rows=normalize)
        dm.ctx.sync()
        res.append(plan.timing())
    tot, steps, launches = min(res[1:] or res, key=lambda t: t[0])
    L = len(coeffs) - 1
    return tot, steps / L, launches, plan  # K1 time per recurrence step (all its launches)


def report(name, S_nnz, n, d, L, dtype, tot, k1, extra):
    es = 8 if dtype == "f64" else 4
    B = S_nnz * (4 + es) + 5 * n * d * es
    line = {"config": name, "dtype": dtype, "n": n, "nnz": S_nnz, "d": d, "L": L,
            "embed_ms": round(tot, 3), "k1_ms_per_step": round(k1, 4),
            "nnz_d_L_per_s": S_nnz * d * L / (tot * 1e-3),
            "k1_step_algorithmic_GBps": round(B / (k1 * 1e-3) / 1e9, 1), "k1_step_frac_of_measured_hbm": round(B / (k1 * 1e-3) / 1e9 / PEAK, 4),
            "algorithmic_bytes_per_step": B, "gather_bytes_per_step": S_nnz * d * es, **extra}
    print(json.dumps(line), flush=True)


def config3(args):
    t0 = time.perf_counter()
    e = db.chung_lu_edges(10_000_000, seed=3)
    A = db.normalized_adjacency(e, 10_000_000)
    del e
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    deg = (A.row_offsets[1:] - A.row_offsets[:-1])
    maxdeg = int(deg.max())
    for dt in args.dtype.split(","):
        dm = A.to_device_matrix("float64" if dt == "f64" else "float32")
        coeffs = pb.legendre_coefficients(pb.commute_time(0.01), 180).coeffs
        tot, k1, launches, plan = run_embed(dm, coeffs, 80, args.reps, dt)
        report("config3 Chung-Lu n=1e7", A.nnz, A.n_rows, 80, 180, dt, tot, k1,
               {"device_build_s": round(build, 2), "max_degree": maxdeg, "k1_launches_per_step": launches / 180})
        dm.close()


def config4(args):
    t0 = time.perf_counter()
    A = db.bag_of_words(2_000_000, 500_000, seed=4)
    S = db.dilate(A)
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    N = S.n_rows
    k = max(1, math.ceil(6.0 * math.log(N)))
    f = pb.odd_extension(CutAbove(0.3))
    coeffs = pb.legendre_coefficients(f, 120).coeffs
    for dt in args.dtype.split(","):
        dm = S.to_device_matrix("float64" if dt == "f64" else "float32")
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        est = dm.spectral_norm(30, k, pb.fold_seed(4, pb.engine.NORM_SEED_TAG), 1.01)
        norm_s = time.perf_counter() - t1
        dm.scale(1.0 / est)
        tot, k1, launches, plan = run_embed(dm, coeffs, 96, args.reps, dt)
        # the split of fast_embed_general: first n rows embed A's columns, last m its rows
        report("config4 BoW 2e6x5e5 dilation", S.nnz, N, 96, 120, dt, tot, k1,
               {"device_build_s": round(build, 2), "A_nnz": A.nnz, "norm_estimate": est,
                "norm_30_iters_k": k, "norm_s": round(norm_s, 3), "k1_launches_per_step": launches / 120})
        dm.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--row-order", type=int, default=None)
    args = ap.parse_args()
    ROW_ORDER = args.row_order
    for c in args.configs.split(","):
        {"3": config3, "4": config4}[c](args)
        torch.cuda.empty_cache()
