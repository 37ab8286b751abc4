"""pytest plugin: the reference's own test suite with the device seam installed.

    PYTHONPATH=baseline/_ref:baseline/_ref/tests:tools:. \
        python -m pytest -p ref_suite_plugin baseline/_ref/tests

`pb.install(csemb)` rebinds the reference's seam (engine._apply_expansion,
sample_projection, estimate_spectral_norm) and downstream consumers
(cluster.kmeans / modularity, oracle._pair_correlations) to this package's
device path before any test runs, so every embedding the reference's tests
compute runs through libcsemb_cuda.so on the GPU.  The session summary counts
the device calls (CSEMB_REF_SUITE_CALLS=1 prints them).
"""

import collections

CALLS = collections.Counter()


def pytest_configure(config):
    import csemb

    import paper_1509_08360_b200 as pb
    from paper_1509_08360_b200 import engine

    pb.install(csemb)
    # One tiny embedding before the suite: CUDA context creation, the library's
    # module load and its first kernel launches (~1.5 s once per process) would
    # otherwise be charged to whichever test runs first -- A1, whose own
    # wall-clock bound is 1 s (test_acceptance.py:52-56).
    import numpy as np

    warm = csemb.SparseMatrix.from_dense(np.eye(4))
    csemb.fast_embed_eig(warm, lambda x: x, 2, csemb.sample_projection(4, 2, seed=0))
    # count how often the reference's code reached the device seam
    for mod in (csemb.engine, getattr(csemb, "oracle", None)):
        if mod is None or not hasattr(mod, "_apply_expansion"):
            continue
        fn = mod._apply_expansion

        def counted(*a, _fn=fn, **k):
            CALLS["_apply_expansion"] += 1
            return _fn(*a, **k)

        mod._apply_expansion = counted
    assert engine is not None


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"device seam calls: {dict(CALLS)}")
