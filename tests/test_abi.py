"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
header declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "csemb_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(csemb_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1509_08360_b200.build import build

    return build()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ["csemb_apply_expansion", "csemb_plan_run", "csemb_matrix_upload", "csemb_spectral_norm",
              "csemb_sample_projection", "csemb_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_1509_08360_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure(lib_path):
    from paper_1509_08360_b200 import _lib
    from paper_1509_08360_b200.errors import CudaUnavailableError

    lib = _lib.load()
    assert lib.csemb_abi_version() == 1
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(CudaUnavailableError):
        _lib.Context(0)
    import paper_1509_08360_b200 as pb

    with pytest.raises(CudaUnavailableError):
        pb.fast_embed_eig(pb.SparseMatrix.identity(4), pb.identity(), 1, pb.SparseMatrix.identity(4).to_dense())


def test_invalid_arguments_return_codes(lib_path):
    from paper_1509_08360_b200 import _lib

    lib = _lib.load()
    assert lib.csemb_ctx_create(0, None) == _lib.ERR_INVALID
    assert b"null" in lib.csemb_last_error()
    assert lib.csemb_plan_run(None, None, 0, 1, None, 0, 0, 0, 1, 0) == _lib.ERR_INVALID
