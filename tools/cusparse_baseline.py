"""Library baseline for K1: cuSPARSE SpMM (torch.sparse CSR on CUDA) plus a
separate elementwise epilogue, on the config-2 workload.

    python tools/cusparse_baseline.py [--dtype f64,f32] [--L 20]

One recurrence step of the baseline = Y = S @ Q(r-1) (cuSPARSE SpMM),
Q(r) = alpha*Y - beta*Q(r-2), E += theta*Q(r) (torch elementwise kernels).
Timed with CUDA events over L steps after warm-up; printed beside the fused
K1 time of the same graph (paper_1509_08360_b200, csemb_plan_run).  The
baseline is not bit-identical to the reference (cuSPARSE's summation order).
"""

import argparse
import json
import os
import sys
import warnings

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64,f32")
ap.add_argument("--L", type=int, default=20)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=80)
ap.add_argument("--config", type=int, default=2, help="2: SBM (host-built); 3 / 4: full-scale device-built inputs")
args = ap.parse_args()
warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")

dev = torch.device("cuda:0")
if args.config == 2:
    S = graphs.sbm(args.n, 100, 15.0, 5.0, seed=2)
    crow, col = torch.from_numpy(S.row_offsets), torch.from_numpy(S.col_indices)
    val = torch.from_numpy(S.values)
else:
    from paper_1509_08360_b200 import device_build as db

    if args.config == 3:
        S = db.normalized_adjacency(db.chung_lu_edges(10_000_000, seed=3), 10_000_000)
    else:
        S = db.dilate(db.bag_of_words(2_000_000, 500_000, seed=4))
        S.values.mul_(1.0 / 130.35983614177252)  # the 30-iteration norm estimate (profiles/r1_configs34.json)
        args.d = 96
    crow, col, val = S.row_offsets, S.col_indices, S.values
    args.n = S.n_rows
coeffs = pb.legendre_coefficients(pb.indicator_above(0.95), args.L).coeffs
out = []
for dt in args.dtype.split(","):
    tdt = torch.float64 if dt == "f64" else torch.float32
    # int32 offsets and column ids (the narrower cuSPARSE index type, like K1's int32 columns)
    A = torch.sparse_csr_tensor(crow.to(dev, torch.int32), col.to(dev, torch.int32), val.to(dev, tdt),
                                size=(S.n_rows, S.n_cols))
    q_prev = torch.randn(args.n, args.d, device=dev, dtype=tdt)
    q_prev2 = torch.randn(args.n, args.d, device=dev, dtype=tdt)
    E = torch.zeros(args.n, args.d, device=dev, dtype=tdt)

    def steps(L, split=None):
        global q_prev, q_prev2
        for r in range(1, L + 1):
            if split is not None:
                split[0].record()
            Y = torch.sparse.mm(A, q_prev)
            if split is not None:
                split[1].record()
            q = Y.mul_(2.0 - 1.0 / r).sub_(q_prev2, alpha=1.0 - 1.0 / r)
            E.add_(q, alpha=float(coeffs[r]))
            q_prev2, q_prev = q_prev, q

    steps(3)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    steps(args.L)
    ev[1].record()
    torch.cuda.synchronize()
    base_ms = ev[0].elapsed_time(ev[1]) / args.L
    sp = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    steps(1, sp)
    torch.cuda.synchronize()
    spmm_ms = sp[0].elapsed_time(sp[1])
    # the fused K1 on the same graph
    dm = pb.DeviceMatrix(S, "float64" if dt == "f64" else "float32") if args.config == 2 else \
        S.to_device_matrix("float64" if dt == "f64" else "float32")
    plan = dm.plan(args.d)
    for _ in range(2):
        plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7)
        dm.ctx.sync()
    _, k1_tot, launches = plan.timing()
    k1_ms = k1_tot / args.L
    dm.close()
    line = {"config": args.config, "dtype": dt, "n": args.n, "nnz": S.nnz, "d": args.d, "cusparse_step_ms": round(base_ms, 4),
            "cusparse_spmm_ms": round(spmm_ms, 4), "fused_k1_ms": round(k1_ms, 4),
            "fused_speedup": round(base_ms / k1_ms, 2)}
    print(json.dumps(line), flush=True)
    out.append(line)
    del A, q_prev, q_prev2, E
    torch.cuda.empty_cache()
