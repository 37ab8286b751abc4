"""Parity checks run in a fresh process by test_gpu_variants.py.

The library reads its experiment switches (CSEMB_K1_TMA, CSEMB_HEAVY_WINDOW_MB,
CSEMB_HOT_ROWS, ...) once per process, so every kernel / schedule variant that
can be selected at run time gets its own process here.  Same checker as the
rest of the GPU suite: the C oracle and the reference's golden config-1 output.
Prints "VARIANT_OK" on success.
"""

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_1509_08360_b200 as pb  # noqa: E402
from conftest import load_golden, sparse_from  # noqa: E402
from paper_1509_08360_b200 import _lib, graphs  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_embed(S, coeffs, om):
    out, _, bad = O.run_stage(O.CSR.of(S), coeffs, om)
    assert bad == 0
    return out


def main():
    _lib.load()
    assert _lib.device_count() > 0
    # config 1: fp64 is the reference's own output bit for bit, fp32 within the gate
    z, meta = load_golden("config1")
    S = sparse_from(z)
    emb = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), pb.EmbedConfig(L=60, d=40, seed=0))
    assert hashlib.sha256(emb.values.tobytes()).hexdigest() == meta["E_sha256"], "config 1 fp64 differs"
    e32 = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), pb.EmbedConfig(L=60, d=40, seed=0), dtype="float32").values
    assert rel(e32, emb.values) <= 1e-4
    # mid-size SBM at the bench's width: fp64 bit-exact against the oracle, fp32 gate
    S = graphs.sbm(30000, 10, 15.0, 5.0, seed=7)
    om = O.sample_projection(30000, 80, 7)
    th = pb.legendre_coefficients(pb.indicator_above(0.95), 24).coeffs
    ref = oracle_embed(S, th, om)
    assert np.array_equal(pb.fast_embed_eig(S, pb.LegendreExpansion(th), 24, om).values, ref), "sbm fp64 differs"
    assert rel(pb.fast_embed_eig(S, pb.LegendreExpansion(th), 24, om, dtype="float32").values, ref) <= 1e-4
    # hub row of 59999 entries over random edges: split rows (chunks / windows / hot pieces),
    # three tile widths, both dtypes; the split changes only the hub row's summation order
    n = 60000
    rng = np.random.default_rng(11)
    e = np.concatenate([np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1), rng.integers(0, n, size=(120000, 2))])
    S = pb.normalized_adjacency(e, n)
    th = pb.legendre_coefficients(pb.commute_time(0.01), 6).coeffs
    dm, dm32 = pb.DeviceMatrix(S), pb.DeviceMatrix(S, "float32")
    for d in (40, 96, 180):
        om = O.sample_projection(n, d, d)
        ref = oracle_embed(S, th, om)
        plan = dm.plan(d)
        got = plan.apply(th, 1, om)
        assert rel(got, ref) <= 1e-13, (d, rel(got, ref))
        assert np.array_equal(plan.apply(th, 1, om), got), d
        assert rel(dm32.plan(d).apply(th, 1, om), ref) <= 1e-4, d
    dm.close()
    dm32.close()
    # power-law graph, strict stored order (no split): bit-exact whatever the variant
    e = graphs.chung_lu_edges(20000, seed=5)
    S = pb.normalized_adjacency(e, 20000)
    om = O.sample_projection(20000, 24, 1)
    th = pb.legendre_coefficients(pb.commute_time(0.01), 15).coeffs
    ref = oracle_embed(S, th, om)
    dm = pb.DeviceMatrix(S)
    plan = dm.plan(24)
    plan.set_load_balance(split_threshold=0)
    assert np.array_equal(plan.apply(th, 1, om), ref), "power-law fp64 differs"
    plan.set_load_balance(split_threshold=64)
    assert rel(plan.apply(th, 1, om), ref) <= 1e-13
    dm.close()
    # banded matrix, 320 entries per row within +-160 columns: over the windowed split
    # threshold when CSEMB_HEAVY_WINDOW_MB is tiny, but every row's entries fall in one
    # or two windows, so the schedule sends them back to the light rows -- strict
    # stored order, bit-exact in every variant
    n = 30000
    base = np.arange(n, dtype=np.int64)
    e = np.concatenate([np.stack([base, (base + k) % n], 1) for k in range(1, 161)])
    S = pb.normalized_adjacency(e, n)
    om = O.sample_projection(n, 16, 9)
    th = pb.legendre_coefficients(pb.indicator_above(0.5), 4).coeffs
    ref = oracle_embed(S, th, om)
    assert np.array_equal(pb.fast_embed_eig(S, pb.LegendreExpansion(th), 4, om).values, ref), "band fp64 differs"
    assert rel(pb.fast_embed_eig(S, pb.LegendreExpansion(th), 4, om, dtype="float32").values, ref) <= 1e-4
    print("VARIANT_OK")


if __name__ == "__main__":
    main()
