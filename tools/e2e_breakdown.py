"""Where the end-to-end (host CSR in, host E out) time of config 2 goes.

    python tools/e2e_breakdown.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import _lib, graphs  # noqa: E402

S = graphs.sbm(1_000_000, 100, 15.0, 5.0, seed=2)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
keep = [pin(S.row_offsets), pin(S.col_indices), pin(S.values)]
ro, ci, va = (t.numpy() for t in keep)
f = pb.indicator_above(0.95)
n, d, L = S.n_rows, 80, 180


def tick(t0, what, acc):
    torch.cuda.synchronize()
    t = time.perf_counter()
    acc.setdefault(what, []).append(1e3 * (t - t0))
    return t


for it in range(5):
    acc = {}
    t = time.perf_counter()
    Sk = pb.SparseMatrix(n, n, ro, ci, va, check=False)
    dm = pb.DeviceMatrix(Sk, "float64")
    t = tick(t, "upload", acc)
    plan = dm.plan(d)
    t = tick(t, "plan_create", acc)
    th = pb.legendre_coefficients(f, L).coeffs
    t = tick(t, "coefficients", acc)
    plan.run(th, 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=7, normalize_rows=True)
    dm.ctx.sync()
    t = tick(t, "run (incl. schedule build)", acc)
    tot, steps, _ = plan.timing()
    out = _lib.host_empty((n, d))
    t = tick(t, "host_empty", acc)
    out2 = plan.download()
    t = tick(t, "download", acc)
    dm.close()
    t = tick(t, "close", acc)
    print(it, {k: round(v[0], 2) for k, v in acc.items()}, "device run", round(tot, 2), flush=True)
