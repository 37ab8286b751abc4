"""Downstream consumers at config-2 scale on one B200.

    python tools/bench_downstream.py [--K 100] [--L 180] [--runs 1] [--out profiles/r1_downstream.json]

Workload: the config-2 SBM (n = 1e6, 100 blocks; host generator, as bench.py), its fp64
embedding (d = 80, L = 180, f = 1{x >= 0.95}, the bench workload) left in HBM,
then on the device-resident E:
  * k-means, K clusters (100 = the SBM's block count), the reference's seeding
    and Lloyd loop (cluster.py:59-107) -- wall time per ++ step and per Lloyd
    iteration, split into assign (K8) and the centroid update (K9);
  * modularity counts over the graph's CSR pattern (K10);
  * cosines of 1e5 sampled row pairs (K5).
Roofline of K8: algorithmic flops 2*n*K*d per assignment (a multiply and an
add per (row, centroid, column)) against the FP64 CUDA-core ceiling measured
by tools/fp64peak.cu (DMUL+DADD pairs, the instruction mix K8 issues).
CPU baseline: the oracle's numpy restatement (the reference's arithmetic,
multithreaded BLAS) on the same rows: one Lloyd iteration and one ++ step.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import cluster as pcl  # noqa: E402
from paper_1509_08360_b200 import distortion as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--K", type=int, default=100)
ap.add_argument("--L", type=int, default=180)
ap.add_argument("--max-iters", type=int, default=100)
ap.add_argument("--fp64-peak", type=float, default=None, help="TFLOP/s (dmul+dadd) from tools/fp64peak")
ap.add_argument("--cpu", type=int, default=1, help="time the numpy baseline too")
ap.add_argument("--out", default=None)
args = ap.parse_args()

res = {"workload": f"config2 SBM n={args.n} d=80 L={args.L} fp64 embedding -> k-means K={args.K}"}
t0 = time.perf_counter()
from paper_1509_08360_b200 import graphs  # noqa: E402

S = graphs.sbm(args.n, 100, 15.0, 5.0, seed=2)  # host generator, as bench.py (config 2)
dm = pb.DeviceMatrix(S, "float64")
dm.ctx.sync()
res["graph_build_s"] = round(time.perf_counter() - t0, 3)
n = dm.n_rows
coeffs = pb.legendre_coefficients(pb.indicator_above(0.95), args.L).coeffs
plan = dm.plan(80)
plan.run(coeffs, 1, omega_kind=pb._lib.OMEGA_SPLITMIX, seed=0)
dm.ctx.sync()
res["embed_ms"] = round(plan.timing()[0], 2)
rows = pcl.plan_rows(plan)

km = pcl.DeviceKMeans(rows, args.K)
# ++ seeding, timed per step (each step: distance to the new centroid, running
# min, fixed-order total, weighted pick) -- the reference's draw sequence
rng = np.random.default_rng(0x6B6D6531)
t = time.perf_counter()
total = km.seed(0, int(rng.integers(n)))
for k in range(1, args.K):
    pick = int(rng.integers(n)) if total <= 0.0 else km.pick(float(rng.random()))
    total = km.seed(k, pick)
seed_s = time.perf_counter() - t
res["pp_seed_ms_per_step"] = round(1e3 * seed_s / args.K, 4)

assign_ms, update_ms, hist = [], [], []
for it in range(args.max_iters):
    t = time.perf_counter()
    inertia, changed, counts = km.assign()
    assign_ms.append(1e3 * (time.perf_counter() - t))
    hist.append(inertia)
    if (counts == 0).any():
        for c in np.flatnonzero(counts == 0):
            km.reseed(int(c))
        km.commit(False)
        continue
    if changed == 0:
        km.commit(False)
        break
    t = time.perf_counter()
    km.commit(True)
    dm.ctx.sync()
    update_ms.append(1e3 * (time.perf_counter() - t))
res["lloyd_iters"] = len(hist)
res["assign_ms_median"] = round(float(np.median(assign_ms)), 4)
res["update_ms_median"] = round(float(np.median(update_ms)), 4) if update_ms else None
flops = 2.0 * n * args.K * 80
res["assign_tflops"] = round(flops / (res["assign_ms_median"] * 1e-3) / 1e12, 3)
if args.fp64_peak:
    res["assign_roofline"] = {"bound": "fp64", "achieved": res["assign_tflops"], "peak": args.fp64_peak,
                              "unit": "TFLOP/s", "frac": round(res["assign_tflops"] / args.fp64_peak, 3),
                              "peak_source": "tools/fp64peak dmul+dadd"}
res["inertia_first_last"] = [hist[0], hist[-1]]
labels_ptr = km.labels_device()
k = int(km.labels().max()) + 1
t = time.perf_counter()
intra, degsum = pcl.modularity_counts(dm, labels_ptr, k)
res["modularity_ms"] = round(1e3 * (time.perf_counter() - t), 3)
res["modularity_Q"] = pcl._score(intra, degsum, dm.nnz // 2).Q

pairs = D.sample_pairs(n, 100_000, 1)
D.pair_correlations(rows, pairs[:1000])
pc = []
for _ in range(5):
    t = time.perf_counter()
    cos, zero = D.pair_correlations(rows, pairs)
    pc.append(1e3 * (time.perf_counter() - t))
res["pair_cos_ms_1e5"] = [round(v, 3) for v in pc]

if args.cpu:
    from oracle.oracle import _sqdist

    E = plan.download()
    C = km.centroids()
    t = time.perf_counter()
    d2 = _sqdist(E, C)
    new = np.argmin(d2, axis=1)
    best = d2[np.arange(n), new]
    float(best.sum())
    acc = np.zeros_like(C)
    np.add.at(acc, new, E)
    res["cpu_lloyd_iter_s"] = round(time.perf_counter() - t, 3)
    t = time.perf_counter()
    _sqdist(E, C[:1])
    res["cpu_pp_step_s"] = round(time.perf_counter() - t, 4)
    res["cpu_threads"] = len(os.sched_getaffinity(0))
    res["cpu_kind"] = "port (oracle numpy restatement of cluster.py, BLAS threads = all cores)"
    res["speedup_lloyd_iter"] = round(res["cpu_lloyd_iter_s"] * 1e3 / (res["assign_ms_median"] + (res["update_ms_median"] or 0)), 1)
km.close()
print(json.dumps(res))
if args.out:
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
