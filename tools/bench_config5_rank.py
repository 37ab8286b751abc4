"""Config 5 (row-partitioned) at full scale, one rank's share, on one B200.

    python tools/bench_config5_rank.py [--gpus 8] [--steps 6] [--dtype f32]

BASELINE config 5: SBM n = 2e8, 2000 blocks, average degree 16, d = 64, L = 100,
fp32, rows partitioned over P GPUs.  Rank 0 of P holds rows
[0, n/P) with GLOBAL column ids and a replicated full Q(r-1) (n x 64 fp32 =
51.2 GB); each step gathers from it (csemb_plan_partition / begin / step,
the same ABI distributed.embed_row_partitioned drives with NCCL).

Measured here: the rank's K1 step time at true scale (CUDA events on the
library stream).  Not measurable on one GPU: the per-step all-gather that
refreshes the full buffer -- reported as its byte count per GPU,
(P-1)/P * n * d * 4 bytes, and the time it takes at an assumed NVLink
all-gather bandwidth (--nvlink-gbs, default 600 GB/s per GPU, not measured).

Synthetic rows (device generator, seeded): Poisson(12) intra-block neighbours
uniform in the row's block of 1e5 rows, Poisson(4) inter-block neighbours
uniform over all n rows, columns sorted per row, values 1/16.  Timing does not
depend on the values; the stored-order arithmetic is the same as any run.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib  # noqa: E402

_mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
PEAK = json.load(open(_mp))["hbm_gbs"] if os.path.exists(_mp) else 6650.0  # B200_PROFILING.md fallback

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000_000)
ap.add_argument("--gpus", type=int, default=8)
ap.add_argument("--block", type=int, default=100_000)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--nvlink-gbs", type=float, default=600.0)
ap.add_argument("--out", default=None)
ap.add_argument("--split", action="store_true",
                help="also time the split exchange (csemb_plan_partition_split): the local-column part "
                     "that overlaps the all-gather, and the remote part + epilogue that follows it")
args = ap.parse_args()

dev = torch.device("cuda:0")
n, P, d = args.n, args.gpus, args.d
nloc = (n + P - 1) // P
g = torch.Generator(device=dev)
g.manual_seed(5)
t0 = time.perf_counter()
rows = torch.arange(nloc, device=dev, dtype=torch.int64)
k_in = torch.poisson(torch.full((nloc,), 12.0, device=dev), generator=g).to(torch.int64)
k_out = torch.poisson(torch.full((nloc,), 4.0, device=dev), generator=g).to(torch.int64)
deg = k_in + k_out
rowptr = torch.zeros(nloc + 1, dtype=torch.int64, device=dev)
rowptr[1:] = torch.cumsum(deg, 0)
nnz = int(rowptr[-1])
# entry -> row, then intra-block or global target
owner = torch.repeat_interleave(rows, deg)
pos = torch.arange(nnz, device=dev, dtype=torch.int64) - rowptr[owner]
intra = pos < k_in[owner]
del pos
blk0 = (owner // args.block) * args.block
u = torch.rand(nnz, device=dev, generator=g, dtype=torch.float32)
cols = torch.where(intra, blk0 + (u * args.block).to(torch.int64).clamp_(max=args.block - 1),
                   (u.double() * n).to(torch.int64).clamp_(max=n - 1))
del u, intra, blk0
# sort columns within each row (stored order = ascending column, like a CSR builder)
key = owner * n + cols
del owner
key, _ = torch.sort(key)
cols = (key % n).to(torch.int32)
del key
torch.cuda.synchronize()
build_s = time.perf_counter() - t0
vdt = torch.float32 if args.dtype == "f32" else torch.float64
vals = torch.full((nnz,), 1.0 / 16.0, device=dev, dtype=torch.float64)  # the ABI takes f64 values
dm = pb.DeviceMatrix.from_device(nloc, n, nnz, rowptr.data_ptr(), cols.data_ptr(), 4, vals.data_ptr(),
                                 "float32" if args.dtype == "f32" else "float64")
del vals, cols
torch.cuda.empty_cache()
plan = dm.plan(d)
_, ld, _ = plan.output()
full = torch.empty((n, ld), device=dev, dtype=vdt)  # the replicated Q(r-1)
q0 = torch.empty((nloc, ld), device=dev, dtype=vdt)
q1 = torch.empty((nloc, ld), device=dev, dtype=vdt)
plan.partition(0, n, full.data_ptr(), q0.data_ptr(), q1.data_ptr())
coeffs = pb.legendre_coefficients(pb.indicator_above(0.95), 100).coeffs
plan.begin(coeffs, omega_kind=_lib.OMEGA_PHILOX, seed=7)   # writes the full Q(0) (no exchange before step 1)
ext = torch.cuda.ExternalStream(dm.ctx.stream, device=dev)
for r in (1, 2):  # warm-up steps (caches, schedule)
    plan.step(r)
dm.ctx.sync()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(ext)
for r in range(3, 3 + args.steps):
    plan.step(r)  # the exchange that would refresh `full` between steps is not run here
ev1.record(ext)
dm.ctx.sync()
step_ms = ev0.elapsed_time(ev1) / args.steps
es = 4 if args.dtype == "f32" else 8
B = nnz * (4 + es) + 5 * nloc * d * es
ag_bytes = (P - 1) / P * n * d * es
res = {
    "workload": f"config5 SBM n={n} (2000 blocks, deg 16), d={d}, {args.dtype}, rank 0 of {P} (rows [0, {nloc}))",
    "local_rows": nloc, "local_nnz": nnz, "device_build_s": round(build_s, 2),
    "k1_step_ms": round(step_ms, 3),
    "k1_nnz_d_per_s": nnz * d / (step_ms * 1e-3),
    "k1_algorithmic_gbs": round(B / (step_ms * 1e-3) / 1e9, 1),
    "k1_frac_of_measured_hbm": round(B / (step_ms * 1e-3) / 1e9 / PEAK, 3),
    "allgather_bytes_per_gpu_per_step": ag_bytes,
    "allgather_ms_at_assumed_gbs": round(ag_bytes / (args.nvlink_gbs * 1e9) * 1e3, 1),
    "assumed_nvlink_allgather_gbs": args.nvlink_gbs,
    "note": "K1 measured; the all-gather is not measurable on one GPU (byte count and an assumed bandwidth only)",
}
if args.split:
    # SURVEY 8(e) "Overlap": the local-column entries run while the all-gather of
    # Q(r-1) is in flight; only the remote part + the epilogue wait for it
    plan.partition_split(0, n, full.data_ptr(), q0.data_ptr(), q1.data_ptr())
    plan.begin(coeffs, omega_kind=_lib.OMEGA_PHILOX, seed=7)
    for r in (1, 2):
        plan.step_local(r)
        plan.step(r)
    dm.ctx.sync()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    evs[0].record(ext)
    for i, r in enumerate(range(3, 3 + args.steps)):
        plan.step_local(r)
        evs[2 * i + 1].record(ext)
        plan.step(r)
        evs[2 * i + 2].record(ext)
    dm.ctx.sync()
    loc = sum(evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(args.steps)) / args.steps
    rem = sum(evs[2 * i + 1].elapsed_time(evs[2 * i + 2]) for i in range(args.steps)) / args.steps
    ag = res["allgather_ms_at_assumed_gbs"]
    res["split"] = {
        "local_ms": round(loc, 3), "remote_and_epilogue_ms": round(rem, 3),
        "step_ms_allgather_then_k1_model": round(ag + step_ms, 1),
        "step_ms_split_overlap_model": round(max(ag, loc) + rem, 1),
        "note": "split parts measured; the overlap model takes the all-gather at the assumed bandwidth",
    }
print(json.dumps(res))
if args.out:
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
