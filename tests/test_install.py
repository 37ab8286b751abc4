"""install(): rebinding the reference package's seam to the device path.

Runs only where the reference is importable (this build container); the GPU
box has no /root/reference, so the check is skipped there.  Without a GPU the
rebound seam must fail loudly (CudaUnavailableError: no silent CPU fallback);
after uninstall the reference's CPU path must be back and bit-exact.
"""

import hashlib
import os
import sys

import numpy as np
import pytest

import paper_1509_08360_b200 as pb
from conftest import load_golden

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture
def csemb():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    try:
        import csemb as mod
    finally:
        sys.path.remove(REF)
    return mod


def test_install_routes_seam_to_device(csemb):
    z, meta = load_golden("config1")
    S = csemb.SparseMatrix(2000, 2000, z["row_offsets"], z["col_indices"].astype(np.int64), z["values"])
    omega = csemb.sample_projection(2000, 40, 0)
    restore = pb.install(csemb)
    try:
        assert csemb.engine._apply_expansion is not None
        if pb._lib.device_count() == 0:
            with pytest.raises(pb.CudaUnavailableError):
                csemb.fast_embed_eig(S, csemb.indicator_above(0.9), 60, omega)
        else:  # pragma: no cover - GPU present in this container
            emb = csemb.fast_embed_eig(S, csemb.indicator_above(0.9), 60, omega)
            assert hashlib.sha256(emb.values.tobytes()).hexdigest() == meta["E_sha256"]
    finally:
        restore()
    emb = csemb.fast_embed_eig(S, csemb.indicator_above(0.9), 60, omega)
    assert hashlib.sha256(emb.values.tobytes()).hexdigest() == meta["E_sha256"]


def test_install_patches_every_module(csemb):
    import importlib

    before = {m: getattr(importlib.import_module(f"csemb.{m}"), "_apply_expansion", None) for m in ("engine", "oracle")}
    restore = pb.install(csemb)
    try:
        for m in ("engine", "oracle"):
            assert getattr(importlib.import_module(f"csemb.{m}"), "_apply_expansion") is not before[m]
        assert csemb.sample_projection is not None and csemb.estimate_spectral_norm.__module__ == "paper_1509_08360_b200.engine"
    finally:
        restore()
    for m in ("engine", "oracle"):
        assert getattr(importlib.import_module(f"csemb.{m}"), "_apply_expansion") is before[m]


def test_install_patches_downstream_consumers(csemb):
    import importlib

    cl = importlib.import_module("csemb.cluster")
    orc = importlib.import_module("csemb.oracle")
    before = (cl.kmeans, cl.modularity, orc._pair_correlations)
    restore = pb.install(csemb)
    try:
        assert cl.kmeans is pb.kmeans and cl.modularity is pb.modularity
        assert orc._pair_correlations is not before[2]
        if pb._lib.device_count() == 0:
            with pytest.raises(pb.CudaUnavailableError):
                cl.kmeans(np.eye(4), 2)
    finally:
        restore()
    assert (cl.kmeans, cl.modularity, orc._pair_correlations) == before
