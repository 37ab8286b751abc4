import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    return z, meta


def csr_from(z, prefix=""):
    from oracle import CSR

    p = prefix
    return CSR(int(z[p + "n_rows"]), int(z[p + "n_cols"]), z[p + "row_offsets"], z[p + "col_indices"],
               z[p + "values"])


def sparse_from(z, prefix=""):
    from paper_1509_08360_b200 import SparseMatrix

    p = prefix
    return SparseMatrix(int(z[p + "n_rows"]), int(z[p + "n_cols"]), z[p + "row_offsets"],
                        z[p + "col_indices"], z[p + "values"])


@pytest.fixture(scope="session")
def config1():
    return load_golden("config1")


@pytest.fixture(scope="session")
def small_cases():
    return load_golden("small_cases")


@pytest.fixture(scope="session")
def gpu_lib():
    """Build (if stale) and load the CUDA library; fail loudly without a GPU."""
    from paper_1509_08360_b200 import _lib
    from paper_1509_08360_b200.build import build

    build()
    _lib.load()
    n = _lib.device_count()
    assert n > 0, "no CUDA device visible: GPU tests must run on the B200 box"
    return _lib


# --------------------------------------------------------------------------
# split-order restatement of the row partition's overlapped exchange
# (csemb_plan_partition_split): per row block [lo, hi), the entries with
# columns inside [lo, hi) are summed first (from +0, stored order), the rest
# separately (from +0, stored order), then y = local + remote -- the checker
# for the split exchange, which is not the reference's summation order
# --------------------------------------------------------------------------
def split_csr(S, lo, hi, rows=None):
    """Rows [lo, hi) of S (or the given row range) cut at columns [lo, hi):
    (local part with ids col - lo, remote part with global ids), each an
    oracle CSR in stored order."""
    import oracle as O

    S = O.CSR.of(S)
    offs = S.row_offsets
    r0, r1 = (lo, hi) if rows is None else rows
    lrow, rrow, lcol, rcol, lval, rval = [0], [0], [], [], [], []
    for i in range(r0, r1):
        c = S.col_indices[offs[i]:offs[i + 1]]
        v = S.values[offs[i]:offs[i + 1]]
        m = (c >= lo) & (c < hi)
        lcol.append(c[m] - lo), lval.append(v[m]), rcol.append(c[~m]), rval.append(v[~m])
        lrow.append(lrow[-1] + int(m.sum())), rrow.append(rrow[-1] + int((~m).sum()))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    return (O.CSR(r1 - r0, hi - lo, lrow, cat(lcol, np.int64), cat(lval, np.float64)),
            O.CSR(r1 - r0, S.n_cols, rrow, cat(rcol, np.int64), cat(rval, np.float64)))


def split_order_stage(S, coeffs, block, blocks):
    """engine._run_stage (engine.py:205-228) with the split exchange's per-row
    order: y = spmm(local part, Q(r-1)[lo:hi]) + spmm(remote part, Q(r-1))."""
    import oracle as O

    parts = [(lo, hi) + split_csr(S, lo, hi) for lo, hi in blocks if hi > lo]
    q_prev = np.array(block, dtype=np.float64)
    acc = coeffs[0] * q_prev
    q_prev2 = None
    for r in range(1, len(coeffs)):
        y = np.empty_like(q_prev)
        for lo, hi, Sl, Sr in parts:
            y[lo:hi] = O.spmm(Sl, q_prev[lo:hi]) + O.spmm(Sr, q_prev)
        q = (2.0 - 1.0 / r) * y
        if r > 1:
            q = q - (1.0 - 1.0 / r) * q_prev2
        acc = acc + coeffs[r] * q
        q_prev2, q_prev = q_prev, q
    return acc
