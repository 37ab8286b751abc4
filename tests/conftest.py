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
