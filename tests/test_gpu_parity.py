"""Device path vs the oracle / the reference's golden vectors (B200 only).

fp64 is bit-identical to the reference (strict separately-rounded multiply/add
in stored-entry order); fp32 meets the north_star tolerances: relative
Frobenius error <= 1e-4 vs the fp64 reference and pairwise cosine error
<= 1e-4 on 10^4 sampled row pairs.
"""

import hashlib
import json
import logging
import os

import numpy as np
import pytest

import oracle as O
import paper_1509_08360_b200 as pb
from conftest import csr_from, load_golden, sparse_from
from paper_1509_08360_b200 import _lib, graphs

pytestmark = pytest.mark.gpu

FP32_REL = 1e-4      # north_star: relative Frobenius error in fp32
COS_TOL = 1e-4       # north_star: pairwise cosine error on sampled pairs


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(autouse=True)
def _lib_ready(gpu_lib):
    yield


# --------------------------------------------------------------------------
# config 1 (BASELINE configs[0]) against the reference's own output
# --------------------------------------------------------------------------
class TestConfig1:
    def test_fp64_bit_exact_given_omega(self, config1):
        z, meta = config1
        S = sparse_from(z)
        emb = pb.fast_embed_eig(S, pb.indicator_above(0.9), 60, O.sample_projection(2000, 40, 0))
        assert sha(emb.values) == meta["E_sha256"]
        assert emb.provenance == meta["provenance"]

    def test_fp64_bit_exact_device_omega(self, config1):
        z, meta = config1
        S = sparse_from(z)
        emb = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), pb.EmbedConfig(L=60, d=40, seed=0))
        assert sha(emb.values) == meta["E_sha256"]
        assert emb.provenance["spmv_products"] == 60
        assert emb.provenance["coeffs_sha256"] == meta["provenance"]["coeffs_sha256"]

    def test_step_log_matches_reference(self, config1, caplog):
        z, _ = config1
        S = sparse_from(z)
        with caplog.at_level(logging.DEBUG, logger="csemb.engine"):
            pb.fast_embed_eig(S, pb.indicator_above(0.9), 60, O.sample_projection(2000, 40, 0))
        recs = [r.getMessage() for r in caplog.records if r.getMessage().startswith("stage=")]
        assert len(recs) == 120
        ref = z["step_max_abs"]
        got = np.array([float(m.split("max_abs=")[1]) for m in recs])
        np.testing.assert_allclose(got, ref[:, 2], rtol=1e-12)
        assert recs[0].startswith("stage=1 cols=0+32 r=1 ") and recs[60].startswith("stage=1 cols=32+8 r=1 ")

    def test_fp32_tolerances(self, config1):
        z, _ = config1
        S = sparse_from(z)
        om = O.sample_projection(2000, 40, 0)
        e32 = pb.fast_embed_eig(S, pb.indicator_above(0.9), 60, om, dtype="float32").values
        assert e32.dtype == np.float64
        assert rel(e32, z["E"]) <= FP32_REL
        pairs = z["pairs"]
        err = np.abs(O.pair_cosines(e32, pairs) - O.pair_cosines(z["E"], pairs)).max()
        assert err <= COS_TOL

    def test_row_normalised_output(self, config1):
        z, _ = config1
        S = sparse_from(z)
        om = O.sample_projection(2000, 40, 0)
        for dt, tol in (("float64", 1e-13), ("float32", FP32_REL)):
            got = pb.fast_embed_eig(S, pb.indicator_above(0.9), 60, om, dtype=dt, normalize_rows=True).values
            ref = O.row_normalize(z["E"])
            assert np.abs(got - ref).max() <= tol
            pairs = z["pairs"]
            cos_dev = np.einsum("ij,ij->i", got[pairs[:, 0]], got[pairs[:, 1]])
            assert np.abs(cos_dev - O.pair_cosines(z["E"], pairs)).max() <= COS_TOL

    def test_repeatable(self, config1):
        z, _ = config1
        S = sparse_from(z)
        a = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), pb.EmbedConfig(L=60, d=40)).values
        b = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), pb.EmbedConfig(L=60, d=40)).values
        assert np.array_equal(a, b)


# --------------------------------------------------------------------------
# engine cases from the reference's suite (golden outputs)
# --------------------------------------------------------------------------
class TestEngineCases:
    def test_cascade_b2(self, small_cases):
        z, meta = small_cases
        S = sparse_from(z, "cascade_")
        counter = pb.SpmvCounter()
        emb = pb.fast_embed_cascaded(S, pb.indicator_above(0.98), pb.EmbedConfig(L=180, d=8, b=2, seed=13),
                                     O.sample_projection(80, 8, 13), counter=counter)
        assert np.array_equal(emb.values, z["cascade_E"])
        assert counter.products == 180
        assert emb.provenance == meta["cascade"]["provenance"]

    def test_general_b2(self, small_cases):
        z, meta = small_cases
        A = sparse_from(z, "general_")
        rows, cols = pb.fast_embed_general(A, pb.indicator_above(0.4), pb.EmbedConfig(L=80, d=9, b=2, seed=18))
        assert np.array_equal(rows.values, z["general_rows"])
        assert np.array_equal(cols.values, z["general_cols"])
        assert rows.provenance == meta["general"]["provenance"]

    def test_general_sparse_config4_weight(self, small_cases):
        z, _ = small_cases

        class CutAbove:
            def __call__(self, x):
                x = np.asarray(x, dtype=np.float64)
                return np.where(x >= 0.3, x, 0.0)

            def breakpoints(self):
                return (0.3,)

        A = sparse_from(z, "general2_")
        rows, cols = pb.fast_embed_general(A, CutAbove(), pb.EmbedConfig(L=120, d=24, seed=4))
        assert np.array_equal(rows.values, z["general2_rows"])
        assert np.array_equal(cols.values, z["general2_cols"])
        r32, c32 = pb.fast_embed_general(A, CutAbove(), pb.EmbedConfig(L=120, d=24, seed=4), dtype="float32")
        assert rel(r32.values, z["general2_rows"]) <= FP32_REL

    def test_chunk_crossing_and_logs(self, small_cases, caplog):
        z, _ = small_cases
        S = sparse_from(z, "wide_")
        om = O.sample_projection(50, 70, 10)
        with caplog.at_level(logging.DEBUG, logger="csemb.engine"):
            emb = pb.fast_embed_eig(S, pb.indicator_above(0.0), 12, om, n_workers=4)
        assert np.array_equal(emb.values, z["wide_E"])
        got = sorted((int(m.split(" r=")[1].split()[0]), int(m.split("cols=")[1].split("+")[0]),
                      float(m.split("max_abs=")[1])) for m in (r.getMessage() for r in caplog.records)
                     if m.startswith("stage="))
        ref = z["wide_steps"]
        assert len(got) == len(ref)
        np.testing.assert_allclose(np.array(got)[:, 2], ref[:, 2], rtol=1e-12)

    def test_polynomial_exactness(self, small_cases):
        z, _ = small_cases
        S = sparse_from(z, "poly_")
        coeffs = z["poly_monomial"]
        emb = pb.fast_embed_eig(S, lambda x: np.polynomial.polynomial.polyval(x, coeffs), 5,
                                O.sample_projection(150, 10, 0))
        assert np.array_equal(emb.values, z["poly_E"])

    def test_column_subset_bit_exact(self, small_cases):
        z, _ = small_cases
        S = sparse_from(z, "wide_")
        om = O.sample_projection(50, 70, 10)
        full = pb.fast_embed_eig(S, pb.indicator_above(0.1), 15, om).values
        part = pb.fast_embed_eig(S, pb.indicator_above(0.1), 15, om[:, 30:37]).values
        assert np.array_equal(part, full[:, 30:37])

    def test_divergence(self, small_cases):
        _, meta = small_cases
        S = pb.SparseMatrix.from_dense(10.0 * np.eye(4))
        with pytest.raises(pb.DivergenceError, match=f"r={meta['divergence']['first_bad_r']} "):
            pb.fast_embed_eig(S, pb.identity(), 250, O.sample_projection(4, 2, 0))

    def test_order_zero(self):
        S = pb.SparseMatrix.from_dense(np.diag([0.5, -0.2, 0.1]))
        om = O.sample_projection(3, 3, 7)
        emb = pb.fast_embed_eig(S, pb.constant(2.5), 0, om)
        assert np.array_equal(emb.values, 2.5 * om) and emb.provenance["spmv_products"] == 0

    def test_identity_and_square(self):  # tests/test_engine.py:100-109
        om = O.sample_projection(8, 4, 5)
        assert np.allclose(pb.fast_embed_eig(pb.SparseMatrix.identity(8), pb.identity(), 1, om).values, om,
                           atol=1e-15)
        S = pb.SparseMatrix.from_dense(np.diag([0.5, -0.5]))
        om = O.sample_projection(2, 6, 6)
        assert np.allclose(pb.fast_embed_eig(S, lambda x: x**2, 2, om).values, 0.25 * om, atol=1e-14)

    def test_errors(self):
        with pytest.raises(ValueError):
            pb.fast_embed_eig(pb.SparseMatrix.identity(4), pb.identity(), 1, np.zeros((3, 2)))
        with pytest.raises(ValueError):
            pb.fast_embed_eig(pb.SparseMatrix.zeros(3, 4), pb.identity(), 1, np.zeros((3, 2)))
        with pytest.raises(ValueError):
            pb.fast_embed_eig(pb.SparseMatrix.identity(4), pb.legendre_coefficients(pb.identity(), 3), 2,
                              np.zeros((4, 2)))


# --------------------------------------------------------------------------
# edge cases and larger inputs against the oracle
# --------------------------------------------------------------------------
def _oracle_embed(S, coeffs, om):
    out, _, bad = O.run_stage(O.CSR.of(S), coeffs, om)
    assert bad == 0
    return out


class TestEdgeCases:
    def test_empty_matrix(self):
        S = pb.SparseMatrix.zeros(6, 6)
        om = O.sample_projection(6, 5, 1)
        th = pb.legendre_coefficients(pb.indicator_above(0.5), 10).coeffs
        got = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 10, om).values
        assert np.array_equal(got, _oracle_embed(S, th, om))

    def test_isolated_vertices_and_zero_rows(self):
        S = pb.normalized_adjacency([(0, 1), (1, 2), (5, 6)], 9)  # 3, 4, 7, 8 isolated
        om = O.sample_projection(9, 6, 2)
        th = pb.legendre_coefficients(pb.indicator_above(0.2), 20).coeffs
        ref = _oracle_embed(S, th, om)
        got = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 20, om).values
        assert np.array_equal(got, ref)
        got = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 20, om, normalize_rows=True).values
        assert np.abs(got - O.row_normalize(ref)).max() <= 1e-15
        assert np.all(np.linalg.norm(got, axis=1)[[3, 4, 7, 8]] > 0)  # Omega rows survive theta_0

    @pytest.mark.parametrize("d", [1, 2, 3, 5, 7, 8, 9, 31, 33, 64, 65, 97, 130, 300, 517])
    def test_widths(self, d):
        S = graphs.sbm(700, 5, 8.0, 2.0, seed=d)
        om = O.sample_projection(700, d, d)
        th = pb.legendre_coefficients(pb.indicator_above(0.6), 9).coeffs
        got = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 9, om).values
        assert np.array_equal(got, _oracle_embed(S, th, om))
        g32 = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 9, om, dtype="float32").values
        assert rel(g32, got) <= FP32_REL

    def test_heavy_rows(self):
        # a star plus a random graph: one row with ~all columns, many with few
        n = 5000
        rng = np.random.default_rng(3)
        e = np.concatenate([np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1),
                            rng.integers(0, n, size=(20000, 2))])
        S = pb.normalized_adjacency(e, n)
        om = O.sample_projection(n, 40, 3)
        th = pb.legendre_coefficients(pb.commute_time(0.01), 25).coeffs
        ref = _oracle_embed(S, th, om)
        # default: the 4999-entry row is split into chunks (deterministic, ~1 ulp)
        got = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 25, om).values
        assert rel(got, ref) <= 1e-13
        again = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 25, om).values
        assert np.array_equal(got, again)
        # splitting off: strict stored-order accumulation, bit-exact
        dm = pb.device_matrix(S)
        plan = dm.plan(40)
        plan.set_load_balance(split_threshold=0)
        assert np.array_equal(plan.apply(th, 1, om), ref)
        # a low threshold splits many rows; still within 1e-13
        plan.set_load_balance(split_threshold=8)
        assert rel(plan.apply(th, 1, om), ref) <= 1e-13
        plan.set_load_balance(split_threshold=4096)

    def test_heavy_combine_many_chunks(self):
        # a 59999-entry hub row = 59 chunks of 1024: the combine's unrolled rounds
        # (24 / 12 / 8 chunks in flight for tiles of <= 32 / 64 / 96 vectors) and
        # its remainder loop, for each width class, in both dtypes
        n = 60000
        rng = np.random.default_rng(11)
        e = np.concatenate([np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1),
                            rng.integers(0, n, size=(120000, 2))])
        S = pb.normalized_adjacency(e, n)
        th = pb.legendre_coefficients(pb.commute_time(0.01), 6).coeffs
        dm, dm32 = pb.DeviceMatrix(S), pb.DeviceMatrix(S, "float32")
        for d in (40, 100, 180):  # fp64 tiles of 20 / 50 / 90 vectors
            om = O.sample_projection(n, d, d)
            ref = _oracle_embed(S, th, om)
            plan = dm.plan(d)
            got = plan.apply(th, 1, om)
            assert rel(got, ref) <= 1e-13, d
            assert np.array_equal(plan.apply(th, 1, om), got), d  # deterministic
            assert rel(dm32.plan(d).apply(th, 1, om), ref) <= FP32_REL, d
        dm.close()
        dm32.close()

    def test_row_order_is_bit_identical(self):
        import scipy.sparse as sp  # noqa: F401

        e = graphs.chung_lu_edges(20000, seed=5)
        S = pb.normalized_adjacency(e, 20000)
        om = O.sample_projection(20000, 24, 1)
        th = pb.legendre_coefficients(pb.commute_time(0.01), 15).coeffs
        ref = _oracle_embed(S, th, om)
        dm = pb.DeviceMatrix(S)
        plan = dm.plan(24)
        plan.set_load_balance(split_threshold=0, row_order=1)
        assert np.array_equal(plan.apply(th, 1, om), ref)
        plan.set_load_balance(row_order=0)
        assert np.array_equal(plan.apply(th, 1, om), ref)
        for ro in (2, 64, 1000, 8192):  # windowed bucketing (auto window / explicit windows)
            plan.set_load_balance(row_order=ro)
            assert np.array_equal(plan.apply(th, 1, om), ref), ro
        with pytest.raises(ValueError):
            plan.set_load_balance(row_order=3)
        plan.set_load_balance(split_threshold=64, row_order=-1)
        got = plan.apply(th, 1, om)
        assert rel(got, ref) <= 1e-13
        g32 = pb.DeviceMatrix(S, "float32").plan(24)
        g32.set_load_balance(split_threshold=64)
        assert rel(g32.apply(th, 1, om), ref) <= FP32_REL
        dm.close()

    def test_norm_with_heavy_rows(self):
        n = 6000
        e = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1)
        S = pb.normalized_adjacency(e, n)  # star: ||S|| = 1
        cfg = pb.EmbedConfig(L=1, d=1, seed=2)
        est = pb.estimate_spectral_norm(S, cfg)
        assert est == pytest.approx(O.spectral_norm(O.CSR.of(S), 2), rel=1e-12)

    def test_midsize_sbm_fp64_fp32(self):
        S = graphs.sbm(30000, 10, 15.0, 5.0, seed=7)
        om = O.sample_projection(30000, 80, 7)
        th = pb.legendre_coefficients(pb.indicator_above(0.95), 40).coeffs
        ref = _oracle_embed(S, th, om)
        got = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 40, om).values
        assert np.array_equal(got, ref)
        g32 = pb.fast_embed_eig(S, pb.LegendreExpansion(th), 40, om, dtype="float32").values
        assert rel(g32, ref) <= FP32_REL
        pairs = O.sample_pairs(30000, 10_000, 1)
        assert np.abs(O.pair_cosines(g32, pairs) - O.pair_cosines(ref, pairs)).max() <= COS_TOL


# --------------------------------------------------------------------------
# projection block, norm estimate, scaling
# --------------------------------------------------------------------------
class TestProjectionAndNorm:
    def test_projection_golden(self):
        z, meta = load_golden("omega")
        for n, d, seed in meta["cases"]:
            om = pb.sample_projection(n, d, seed)
            assert np.array_equal(np.packbits(om > 0), z[f"signs_{n}_{d}_{seed}"])
            assert np.array_equal(om, O.sample_projection(n, d, seed))
        full = pb.sample_projection(300, 80, 9)
        assert np.array_equal(pb.sample_projection(300, 80, 9, col0=20, w=17), full[:, 20:37])

    def test_philox_projection(self):
        n, d = 100_000, 64
        om = pb.sample_projection(n, d, 0, kind="philox")
        assert np.all(np.abs(om) == 1.0 / 8.0)
        assert abs(om.mean()) <= 4.0 * (1 / 8.0) / np.sqrt(n * d)
        assert not np.array_equal(om, pb.sample_projection(n, d, 0))

    def test_norm_golden(self):
        z, meta = load_golden("norm")
        for name, m in meta.items():
            S = sparse_from(z, name + "_")
            cfg = pb.EmbedConfig(L=1, d=1, seed=m["seed"], norm_iters=m["norm_iters"])
            est = pb.estimate_spectral_norm(S, cfg)
            assert est == pytest.approx(m["estimate"], rel=1e-12, abs=1e-15), name
            assert est <= 1.01 * m["exact_norm"] + 1e-12

    def test_norm_edge_cases(self):
        assert pb.estimate_spectral_norm(pb.SparseMatrix.zeros(5, 5), pb.EmbedConfig(L=1, d=1)) == 0.0
        assert pb.estimate_spectral_norm(pb.SparseMatrix.identity(10), pb.EmbedConfig(L=1, d=1)) == \
            pytest.approx(1.01, abs=1e-12)
        with pytest.raises(ValueError):
            pb.estimate_spectral_norm(pb.SparseMatrix.zeros(3, 4), pb.EmbedConfig(L=1, d=1))

    def test_norm_config1_and_philox_start(self, config1):
        z, meta = config1
        S = sparse_from(z)
        cfg = pb.EmbedConfig(L=60, d=40, seed=0)
        assert pb.estimate_spectral_norm(S, cfg) == pytest.approx(meta["norm_estimate"], rel=1e-12)
        est = pb.estimate_spectral_norm(S, cfg, start="philox")
        assert 0.99 <= est <= 1.01 + 1e-12  # ||S|| = 1 for a normalized adjacency

    def test_matrix_scale_bit_exact(self, config1):
        z, _ = config1
        S = sparse_from(z)
        dm = pb.DeviceMatrix(S, "float64")
        f = 1.0 / 1.0099999155519637
        dm.scale(f)
        assert np.array_equal(dm.download_values(), S.values * f)
        dm.close()


# --------------------------------------------------------------------------
# device-side input construction vs the host builders
# --------------------------------------------------------------------------
class TestDeviceBuild:
    def test_normalized_adjacency_matches_host(self, config1):
        import torch

        from paper_1509_08360_b200 import device_build as db

        z, meta = config1
        e = torch.as_tensor(z["edges"].astype(np.int64), device="cuda")
        D = db.normalized_adjacency(e, 2000).to_host()
        assert np.array_equal(D.row_offsets, z["row_offsets"])
        assert np.array_equal(D.col_indices, z["col_indices"])
        assert np.array_equal(D.values, z["values"])
        zb, mb = load_golden("builders")
        for i in range(4):
            n = mb[f"adj{i}"]["n"]
            D = db.normalized_adjacency(torch.as_tensor(zb[f"adj{i}_edges"], device="cuda"), n).to_host()
            assert np.array_equal(D.values, zb[f"adj{i}_values"]) and np.array_equal(D.col_indices, zb[f"adj{i}_col_indices"])

    def test_normalized_adjacency_edge_cases(self):
        # the library kernels (csrc/build.cu) against the host builder: host and
        # device edge arrays, duplicates in both orientations, self-loops,
        # isolated vertices, an empty / loops-only edge list, larger random
        # graphs (multi-pass radix sort), the fp32 copy, and range errors
        import torch

        from paper_1509_08360_b200 import device_build as db

        cases = [(np.array([[0, 1], [1, 0], [1, 1], [2, 3], [3, 2], [2, 3]]), 6),
                 (np.zeros((0, 2), dtype=np.int64), 5),
                 (np.array([[4, 4], [0, 0]]), 5)]
        rng = np.random.default_rng(7)
        for n in (1, 2, 1000, 65_537, 300_000):
            cases.append((rng.integers(0, n, size=(4 * n + 3, 2)), n))
        for edges, n in cases:
            H = pb.normalized_adjacency(edges, n)
            for src in (edges, torch.as_tensor(edges, device="cuda")):
                D = db.normalized_adjacency(src, n)
                assert D.nnz == H.nnz
                assert np.array_equal(D.row_offsets.cpu().numpy(), H.row_offsets)
                assert np.array_equal(D.col_indices.cpu().numpy().astype(np.int64), H.col_indices)
                assert np.array_equal(D.values.cpu().numpy(), H.values)
            m32 = D.to_device_matrix("float32")
            assert np.array_equal(m32.download_values(), H.values.astype(np.float32).astype(np.float64))
            m32.close()
        with pytest.raises(ValueError):
            db.normalized_adjacency(np.array([[0, 5]]), 5)
        with pytest.raises(ValueError):
            db.normalized_adjacency(torch.as_tensor([[-1, 2]], device="cuda"), 5)

    def test_dilate_matches_host(self):
        from paper_1509_08360_b200 import device_build as db

        for m, n, seed in ((1, 1, 0), (7, 3, 1), (3000, 500, 2)):
            A = graphs.bag_of_words(m, n, seed=seed, mean_len=5)
            D = db.dilate(db.from_host(A)).to_host()
            H = pb.dilate(A)
            assert np.array_equal(D.row_offsets, H.row_offsets) and np.array_equal(D.col_indices, H.col_indices)
            assert np.array_equal(D.values, H.values)

        A = graphs.bag_of_words(400, 300, seed=3, mean_len=20)
        D = db.dilate(db.from_host(A)).to_host()
        H = pb.dilate(A)
        assert np.array_equal(D.row_offsets, H.row_offsets)
        assert np.array_equal(D.col_indices, H.col_indices)
        assert np.array_equal(D.values, H.values)

    def test_device_matrix_embed_matches(self, config1):
        import torch

        from paper_1509_08360_b200 import device_build as db

        z, meta = config1
        dm = db.normalized_adjacency(torch.as_tensor(z["edges"].astype(np.int64), device="cuda"), 2000).to_device_matrix()
        plan = dm.plan(40)
        out = plan.apply(z["coeffs"], 1, None, omega_kind=1, seed=0)  # reference hash on the device
        assert sha(out) == meta["E_sha256"]
        dm.close()

    def test_generators_shapes(self):
        from paper_1509_08360_b200 import device_build as db

        e = db.chung_lu_edges(20000, seed=1)
        assert abs(2 * e.shape[0] / 20000 - 20.0) < 1.0
        A = db.bag_of_words(500, 800, seed=2, mean_len=30)
        H = A.to_host()
        H._validate()
        rn = np.sqrt(np.bincount(np.repeat(np.arange(500), np.diff(H.row_offsets)), weights=H.values ** 2,
                                 minlength=500))
        assert np.allclose(rn[rn > 0], 1.0)


# --------------------------------------------------------------------------
# row partition (config 5 layout): emulated ranks on one GPU, NCCL driver at ws=1
# --------------------------------------------------------------------------
def test_device_list_column_shards_bit_exact(config1, caplog):
    # device=[0, 0]: two column shards driven concurrently from one process
    # (both on the one GPU here), assembled, optionally K4-normalised
    z, meta = config1
    S = sparse_from(z)
    cfg = pb.EmbedConfig(L=60, d=40, seed=0)
    one = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), cfg).values
    two = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), cfg, device=[0, 0]).values
    assert np.array_equal(one, two)
    assert sha(two) == meta["E_sha256"]
    three = pb.fast_embed_cascaded(S, pb.indicator_above(0.9), cfg, device=[0, 0, 0], normalize_rows=True).values
    assert np.array_equal(three, pb.fast_embed_cascaded(S, pb.indicator_above(0.9), cfg, normalize_rows=True).values)
    om = O.sample_projection(2000, 40, 3)
    th = pb.legendre_coefficients(pb.indicator_above(0.9), 12)
    a = pb.fast_embed_eig(S, th, 12, om, dtype="float32", device=[0, 0]).values
    assert np.array_equal(a, pb.fast_embed_eig(S, th, 12, om, dtype="float32").values)
    # the debug log equals the one-device log (chunk maxima combined over shards)
    with caplog.at_level(logging.DEBUG, logger="csemb.engine"):
        pb.fast_embed_eig(S, th, 12, om, device=[0, 0])
    multi = [r.getMessage() for r in caplog.records if r.getMessage().startswith("stage=")]
    caplog.clear()
    with caplog.at_level(logging.DEBUG, logger="csemb.engine"):
        pb.fast_embed_eig(S, th, 12, om)
    single = [r.getMessage() for r in caplog.records if r.getMessage().startswith("stage=")]
    assert multi == single and len(single) == 24
    # divergence: the first bad step over all shards
    with pytest.raises(pb.DivergenceError) as e1:
        pb.fast_embed_eig(pb.scale_values(S, 1e40), th, 12, om, device=[0, 0])
    with pytest.raises(pb.DivergenceError) as e2:
        pb.fast_embed_eig(pb.scale_values(S, 1e40), th, 12, om)
    assert str(e1.value) == str(e2.value)
    with pytest.raises(ValueError):
        pb.fast_embed_eig(S, th, 12, om, device=[])


class TestRowPartition:
    @pytest.mark.parametrize("dtype", ["float64", "float32"])
    def test_emulated_ranks_bit_exact(self, dtype):
        import torch

        from paper_1509_08360_b200.distributed import local_rows, row_blocks

        S = graphs.sbm(3001, 7, 10.0, 3.0, seed=4)
        n, d, L = S.n_rows, 40, 12
        th = pb.legendre_coefficients(pb.indicator_above(0.5), L).coeffs
        ref = pb.DeviceMatrix(S, dtype).plan(d).apply(th, 1, None, omega_kind=1, seed=3)
        tdt = torch.float64 if dtype == "float64" else torch.float32
        world = 3
        n_pad, blocks = row_blocks(n, world)
        F = torch.zeros((world * n_pad, d), dtype=tdt, device="cuda")
        ranks = []
        for lo, hi in blocks:
            dm = pb.DeviceMatrix(local_rows(S, lo, hi), dtype)
            plan = dm.plan(d)
            q = [torch.zeros((n_pad, d), dtype=tdt, device="cuda") for _ in range(2)]
            plan.partition(lo, n, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
            torch.cuda.synchronize()  # torch's zero-fills before the library stream writes
            plan.begin(th, omega_kind=1, seed=3)
            ranks.append((lo, hi, dm, plan, q))
        for r in range(1, L + 1):
            for lo, hi, dm, plan, q in ranks:  # independent launches: no rank waits on another
                plan.step(r)
            for _, _, dm, _, _ in ranks:
                dm.ctx.sync()
            if r < L:
                for lo, hi, dm, plan, q in ranks:  # the all-gather, emulated by copies
                    F[lo:hi] = q[r & 1][:hi - lo]
                torch.cuda.synchronize()
        got = []
        for lo, hi, dm, plan, q in ranks:
            plan.end(False)
            got.append(plan.download())
            dm.close()
        assert np.array_equal(np.concatenate(got), ref)

    @pytest.mark.parametrize("dtype", ["float64", "float32"])
    def test_split_exchange_emulated(self, dtype):
        # csemb_plan_partition_split: per step every "rank" runs its local-column
        # part from its own Q(r-1) rows, then (after the emulated all-gather) the
        # remote part + epilogue.  fp64: bit-identical to the split-order
        # restatement; both dtypes within rounding of the 1-GPU stored order.
        import torch

        from conftest import split_order_stage
        from paper_1509_08360_b200.distributed import local_rows, row_blocks

        S = graphs.sbm(3001, 7, 10.0, 3.0, seed=4)
        n, d, L = S.n_rows, 40, 12
        th = pb.legendre_coefficients(pb.indicator_above(0.5), L).coeffs
        om = O.sample_projection(n, d, 3)
        tdt = torch.float64 if dtype == "float64" else torch.float32
        world = 3
        n_pad, blocks = row_blocks(n, world)
        F = torch.zeros((world * n_pad, d), dtype=tdt, device="cuda")
        ranks = []
        for lo, hi in blocks:
            dm = pb.DeviceMatrix(local_rows(S, lo, hi), dtype)
            plan = dm.plan(d)
            q = [torch.zeros((n_pad, d), dtype=tdt, device="cuda") for _ in range(2)]
            plan.partition_split(lo, n, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
            torch.cuda.synchronize()
            plan.begin(th, omega_kind=1, seed=3)
            ranks.append((lo, hi, dm, plan, q))
        for r in range(1, L + 1):
            for lo, hi, dm, plan, q in ranks:
                plan.step_local(r)
            for lo, hi, dm, plan, q in ranks:  # F holds Q(r-1) of every rank (emulated all-gather)
                plan.step(r)
            for _, _, dm, _, _ in ranks:
                dm.ctx.sync()
            if r < L:
                for lo, hi, dm, plan, q in ranks:
                    F[lo:hi] = q[r & 1][:hi - lo]
                torch.cuda.synchronize()
        got = []
        for lo, hi, dm, plan, q in ranks:
            plan.end(False)
            got.append(plan.download())
            dm.close()
        got = np.concatenate(got)
        if dtype == "float64":
            assert np.array_equal(got, split_order_stage(O.CSR.of(S), th, om, blocks))
        ref = _oracle_embed(S, th, om)
        assert rel(got, ref) <= (1e-13 if dtype == "float64" else FP32_REL)

    @pytest.mark.parametrize("split_threshold", [0, None])
    def test_split_exchange_heavy_rows(self, split_threshold):
        # a power-law graph plus a 6000-entry hub row: heavy rows in both column
        # parts (chunked SpMM + combine inside each part).  Strict stored order
        # (threshold 0): bit-identical to the split-order restatement; default
        # chunking: within rounding.
        import torch

        from conftest import split_order_stage
        from paper_1509_08360_b200.distributed import local_rows, row_blocks

        rng = np.random.default_rng(0)
        n = 30011
        e = np.concatenate([graphs.chung_lu_edges(n, seed=1),
                            np.stack([np.full(6000, 7, np.int64), rng.integers(0, n, 6000)], 1)])
        S = pb.normalized_adjacency(e, n)
        d, L = 24, 8
        th = pb.legendre_coefficients(pb.commute_time(0.01), L).coeffs
        om = O.sample_projection(n, d, 3)
        world = 3
        n_pad, blocks = row_blocks(n, world)
        F = torch.zeros((world * n_pad, d), dtype=torch.float64, device="cuda")
        ranks = []
        for lo, hi in blocks:
            dm = pb.DeviceMatrix(local_rows(S, lo, hi), "float64")
            plan = dm.plan(d)
            if split_threshold is not None:
                plan.set_load_balance(split_threshold=split_threshold)
            q = [torch.zeros((n_pad, d), dtype=torch.float64, device="cuda") for _ in range(2)]
            plan.partition_split(lo, n, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
            torch.cuda.synchronize()
            plan.begin(th, omega_kind=1, seed=3)
            ranks.append((lo, hi, dm, plan, q))
        for r in range(1, L + 1):
            for *_, plan, _ in ranks:
                plan.step_local(r)
            for *_, plan, _ in ranks:
                plan.step(r)
            for _, _, dm, _, _ in ranks:
                dm.ctx.sync()
            if r < L:
                for lo, hi, dm, plan, q in ranks:
                    F[lo:hi] = q[r & 1][:hi - lo]
                torch.cuda.synchronize()
        got = []
        for lo, hi, dm, plan, q in ranks:
            plan.end(False)
            got.append(plan.download())
            dm.close()
        got = np.concatenate(got)
        if split_threshold == 0:
            assert np.array_equal(got, split_order_stage(O.CSR.of(S), th, om, blocks))
        assert rel(got, _oracle_embed(S, th, om)) <= 1e-13

    def test_split_exchange_needs_local_step(self):
        import torch

        S = graphs.sbm(500, 2, 6.0, 2.0, seed=1)
        dm = pb.DeviceMatrix(S, "float64")
        plan = dm.plan(8)
        F = torch.zeros((500, 8), dtype=torch.float64, device="cuda")
        q = [torch.zeros((500, 8), dtype=torch.float64, device="cuda") for _ in range(2)]
        plan.partition_split(0, 500, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
        torch.cuda.synchronize()
        plan.begin(pb.legendre_coefficients(pb.indicator_above(0.5), 3).coeffs, omega_kind=1, seed=1)
        with pytest.raises(ValueError, match="step_local"):
            plan.step(1)
        dm.close()

    @pytest.mark.parametrize("dtype", ["float64", "float32"])
    def test_fused_peer_exchange_emulated(self, dtype):
        # csemb_plan_partition_peers: each "rank" stores its Q(r) rows into the
        # other ranks' replicated buffers from K1's epilogue (here: buffers on
        # the same GPU standing in for NVLink-mapped peers).  Ranks never wait
        # on one another; the per-step barrier is a host sync of every rank.
        import torch

        from paper_1509_08360_b200.distributed import local_rows, row_blocks

        S = graphs.sbm(3001, 7, 10.0, 3.0, seed=4)
        n, d, L = S.n_rows, 40, 12
        th = pb.legendre_coefficients(pb.indicator_above(0.5), L).coeffs
        ref = pb.DeviceMatrix(S, dtype).plan(d).apply(th, 1, None, omega_kind=1, seed=3)
        tdt = torch.float64 if dtype == "float64" else torch.float32
        world = 3
        n_pad, blocks = row_blocks(n, world)
        F = [[torch.zeros((world * n_pad, d), dtype=tdt, device="cuda") for _ in range(2)] for _ in range(world)]
        torch.cuda.synchronize()
        ranks = []
        for p, (lo, hi) in enumerate(blocks):
            dm = pb.DeviceMatrix(local_rows(S, lo, hi), dtype)
            plan = dm.plan(d)
            others = [q for q in range(world) if q != p]
            plan.partition_peers(lo, n, (F[p][0].data_ptr(), F[p][1].data_ptr()),
                                 [F[q][0].data_ptr() for q in others], [F[q][1].data_ptr() for q in others])
            plan.begin(th, omega_kind=1, seed=3)
            ranks.append((dm, plan))
        for dm, _ in ranks:
            dm.ctx.sync()
        for r in range(1, L + 1):
            for _, plan in ranks:
                plan.step(r)
            for dm, _ in ranks:  # the per-step barrier
                dm.ctx.sync()
        got = []
        for dm, plan in ranks:
            plan.end(False)
            got.append(plan.download())
            dm.close()
        assert np.array_equal(np.concatenate(got), ref)
        # every replica holds the whole final Q(L) (parity L & 1), identical across ranks
        torch.cuda.synchronize()
        for p in range(1, world):
            assert torch.equal(F[p][L & 1][:n], F[0][L & 1][:n])

    @pytest.mark.parametrize("dtype", ["float64", "float32"])
    def test_fused_peer_exchange_emulated_power_law(self, dtype):
        # the fused exchange at scale on a power-law graph: Chung-Lu n = 1e6
        # (device-built), 3 emulated ranks, rows above the split threshold
        # chunked on every rank exactly as on one GPU -- the heavy-row combine
        # kernel stores its Q(r) rows into the peers' replicas too.  Bit-identical
        # to the single-GPU run with the same (default) schedule.
        import torch

        from paper_1509_08360_b200 import device_build as db
        from paper_1509_08360_b200.distributed import row_blocks

        n, d, L, world = 1_000_000, 40, 6, 3
        S = db.normalized_adjacency(db.chung_lu_edges(n, seed=11), n)
        assert int((S.row_offsets[1:] - S.row_offsets[:-1]).max()) > 2048  # split rows present
        th = pb.legendre_coefficients(pb.indicator_above(0.5), L).coeffs
        dm1 = S.to_device_matrix(dtype)
        ref = dm1.plan(d).apply(th, 1, None, omega_kind=1, seed=3)
        dm1.close()
        tdt = torch.float64 if dtype == "float64" else torch.float32
        n_pad, blocks = row_blocks(n, world)
        F = [[torch.zeros((world * n_pad, d), dtype=tdt, device="cuda") for _ in range(2)] for _ in range(world)]
        torch.cuda.synchronize()
        ro, ci, va = S.row_offsets, S.col_indices, S.values
        ranks = []
        for p, (lo, hi) in enumerate(blocks):
            a, b = int(ro[lo]), int(ro[hi])
            part = db.DeviceCSR(hi - lo, n, (ro[lo:hi + 1] - a).contiguous(), ci[a:b].contiguous(),
                                va[a:b].contiguous())
            dm = part.to_device_matrix(dtype)
            plan = dm.plan(d)
            others = [q for q in range(world) if q != p]
            plan.partition_peers(lo, n, (F[p][0].data_ptr(), F[p][1].data_ptr()),
                                 [F[q][0].data_ptr() for q in others], [F[q][1].data_ptr() for q in others])
            plan.begin(th, omega_kind=1, seed=3)
            ranks.append((dm, plan))
        for dm, _ in ranks:
            dm.ctx.sync()
        for r in range(1, L + 1):
            for _, plan in ranks:  # independent launches: no rank waits on another
                plan.step(r)
            for dm, _ in ranks:  # the per-step barrier
                dm.ctx.sync()
        got = []
        for dm, plan in ranks:
            plan.end(False)
            got.append(plan.download())
            dm.close()
        assert np.array_equal(np.concatenate(got), ref)

    def test_fused_peer_exchange_errors(self):
        S = graphs.sbm(500, 2, 6.0, 2.0, seed=1)
        dm = pb.DeviceMatrix(S)
        plan = dm.plan(8)
        import torch

        F = [torch.zeros((500, 8), dtype=torch.float64, device="cuda") for _ in range(2)]
        with pytest.raises(ValueError):
            plan.partition_peers(0, 500, (F[0].data_ptr(), F[1].data_ptr()), [F[0].data_ptr()], [])
        with pytest.raises(ValueError):
            plan.partition_peers(0, 500, (F[0].data_ptr(), F[1].data_ptr()), [0], [0])
        with pytest.raises(ValueError):
            plan.partition_peers(0, 500, (F[0].data_ptr(), F[1].data_ptr()), [F[0].data_ptr()] * 16,
                                 [F[1].data_ptr()] * 16)
        plan.partition_peers(0, 500, (F[0].data_ptr(), F[1].data_ptr()))
        th = pb.legendre_coefficients(pb.indicator_above(0.5), 3).coeffs
        with pytest.raises(NotImplementedError):  # the fused exchange generates Q(0) itself
            plan.begin(th, block_dev=F[0].data_ptr(), omega_kind=0)
        plan.begin(th, omega_kind=1, seed=5)
        for r in range(1, 4):
            plan.step(r)
        plan.end(False)
        ref = pb.DeviceMatrix(S).plan(8).apply(th, 1, None, omega_kind=1, seed=5)
        assert np.array_equal(plan.download(), ref)
        dm.close()

    def test_nccl_driver_world_one(self):
        import socket

        import torch
        import torch.distributed as dist

        from paper_1509_08360_b200.distributed import embed_row_partitioned

        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        try:
            S = graphs.sbm(2000, 4, 8.0, 2.0, seed=6)
            th = pb.legendre_coefficients(pb.indicator_above(0.3), 9).coeffs
            E, peaks = embed_row_partitioned(S, 0, S.n_rows, th, 24, seed=2, device=0)
            ref, _, _ = O.run_stage(O.CSR.of(S), th, O.sample_projection(S.n_rows, 24, 2))
            assert np.array_equal(E.cpu().numpy(), ref)
            assert np.all(np.isfinite(peaks)) and not np.any(peaks >= np.inf)
            # the fused exchange through torch symmetric memory (no peers at world 1)
            E2, _ = embed_row_partitioned(S, 0, S.n_rows, th, 24, seed=2, device=0, exchange="peer")
            assert np.array_equal(E2.cpu().numpy(), ref)
            # the split (overlapped) exchange: at world 1 every column is local, so
            # the order is the stored one: bit-identical too (the all-gather runs on
            # its own stream, ordered by events against the library stream)
            Es, _ = embed_row_partitioned(S, 0, S.n_rows, th, 24, seed=2, device=0, exchange="split")
            assert np.array_equal(Es.cpu().numpy(), ref)
            # C1: the CSR broadcast over NCCL into device memory, then the column-sharded run
            from paper_1509_08360_b200.distributed import broadcast_matrix, embed_column_sharded

            Sd = broadcast_matrix(S, src=0, device=0)
            assert Sd.col_indices.dtype == torch.int32 and Sd.col_indices.is_cuda
            E6, _ = embed_column_sharded(Sd, th, 24, seed=2, device=0, normalize_rows=False)
            assert np.array_equal(E6.cpu().numpy(), ref)
            # K4 after the gather, ordered on the library stream (no host sync in between)
            E7, _ = embed_column_sharded(Sd, th, 24, seed=2, device=0, normalize_rows=True)
            np.testing.assert_allclose(E7.cpu().numpy(), O.row_normalize(ref), rtol=0, atol=1e-15)
            # the 2-D grid driver at 1 x 1 (row partition + column assembly + K4), both exchanges
            from paper_1509_08360_b200.distributed import embed_2d

            for ex in ("allgather", "peer"):
                E4, _ = embed_2d(S, th, 24, (1, 1), seed=2, device=0, exchange=ex, normalize_rows=False)
                assert np.array_equal(E4.cpu().numpy(), ref), ex
            E5, _ = embed_2d(S, th, 24, (1, 1), seed=2, device=0)
            np.testing.assert_allclose(E5.cpu().numpy(), O.row_normalize(ref), rtol=0, atol=1e-15)
            # ... and through NVLS multicast, where the node offers it (multimem.st
            # into the one-replica multicast object)
            try:
                E3, _ = embed_row_partitioned(S, 0, S.n_rows, th, 24, seed=2, device=0, exchange="multicast",
                                              dtype="f64")
            except RuntimeError as e:
                if "multicast is not available" not in str(e):
                    raise
                print("NVLS multicast unavailable here:", e)
            else:
                assert np.array_equal(E3.cpu().numpy(), ref)
        finally:
            dist.destroy_process_group()


# --------------------------------------------------------------------------
# CLI drop-in: the reference's own command lines, outputs compared
# --------------------------------------------------------------------------
class TestCLI:
    def _inputs(self, tmp_path):
        import scipy.io
        import scipy.sparse as sp

        z, meta = load_golden("cli")
        g = tmp_path / "g.txt"
        g.write_text("\n".join(f"{u} {v}" for u, v in z["edges"]) + "\n")
        scipy.io.mmwrite(str(tmp_path / "raw.mtx"), sp.coo_array(z["raw"]))
        scipy.io.mmwrite(str(tmp_path / "rect.mtx"), sp.coo_array(z["rect"]))
        return z, meta

    def _argv(self, meta, name, tmp_path):
        argv = list(meta[name]["argv"])
        i = argv.index("--input")
        argv[i + 1] = str(tmp_path / os.path.basename(argv[i + 1]))
        return argv

    def test_edgelist_byte_identical(self, tmp_path):
        from paper_1509_08360_b200.cli import main

        z, meta = self._inputs(tmp_path)
        out = str(tmp_path / "e.bin")
        assert main(self._argv(meta, "edgelist", tmp_path) + ["--output", out]) == 0
        assert hashlib.sha256(open(out, "rb").read()).hexdigest() == meta["edgelist"]["sha256"]
        md = json.load(open(out + ".meta.json"))
        for k, v in meta["edgelist"]["metadata"].items():
            assert md[k] == v, k

    def test_raw_and_dilation(self, tmp_path):
        from paper_1509_08360_b200 import io as bio
        from paper_1509_08360_b200.cli import main

        z, meta = self._inputs(tmp_path)
        out = str(tmp_path / "r.bin")
        assert main(self._argv(meta, "raw", tmp_path) + ["--output", out]) == 0
        assert rel(bio.read_embedding(out), z["raw_E"]) <= 1e-12
        md = json.load(open(out + ".meta.json"))
        assert md["norm_estimate"] == pytest.approx(meta["raw"]["metadata"]["norm_estimate"], rel=1e-12)
        assert md["spmv_products"] == meta["raw"]["metadata"]["spmv_products"]
        out = str(tmp_path / "d.bin")
        cols = str(tmp_path / "d.cols.bin")
        assert main(self._argv(meta, "dilation", tmp_path) + ["--output", out, "--output-cols", cols]) == 0
        assert rel(bio.read_embedding(out), z["dilation_E"]) <= 1e-12
        assert rel(bio.read_embedding(cols), z["dilation_cols"]) <= 1e-12
        md = json.load(open(out + ".meta.json"))
        assert md["coeffs_sha256"] == meta["dilation"]["metadata"]["coeffs_sha256"]

    def test_norm_command(self, tmp_path, capsys):
        from paper_1509_08360_b200.cli import main

        z, meta = self._inputs(tmp_path)
        assert main(["norm", "--input", str(tmp_path / "raw.mtx"), "--format", "matrix-market", "--matrix", "raw",
                     "--seed", "3"]) == 0
        got = json.loads(capsys.readouterr().out)
        assert got["norm_estimate"] == pytest.approx(meta["norm"]["norm_estimate"], rel=1e-12)


class TestEFold:
    """E is read/written every 3 steps with the pending terms added in the
    reference's order: every L (all flush patterns) stays bit-exact."""

    @pytest.mark.parametrize("L", list(range(0, 9)))
    def test_orders_bit_exact(self, L):
        S = graphs.sbm(1500, 5, 8.0, 2.0, seed=L)
        om = O.sample_projection(1500, 24, L)
        th = np.random.default_rng(L).standard_normal(L + 1) * 0.4
        ref = _oracle_embed(S, th, om)
        for fold in (1, 2, 3):
            plan = pb.device_matrix(S).plan(24)
            plan.set_option(_lib.OPT_E_FOLD, fold)
            assert np.array_equal(plan.apply(th, 1, om), ref), (L, fold)
            plan.set_option(_lib.OPT_E_FOLD, 3)

    def test_cascade_stages(self):
        S = graphs.sbm(1200, 4, 8.0, 2.0, seed=9)
        om = O.sample_projection(1200, 16, 9)
        th = np.random.default_rng(9).standard_normal(8) * 0.4
        ref, _, _ = O.apply_expansion(O.CSR.of(S), th, om, n_stages=3)
        got = pb.device_matrix(S).plan(16).apply(th, 3, om)
        assert np.array_equal(got, ref)


class TestABIErrors:
    """Every invalid request returns CSEMB_ERR_INVALID (ValueError), never a crash."""

    def test_plan_argument_checks(self):
        S = graphs.sbm(300, 3, 6.0, 2.0, seed=1)
        dm = pb.DeviceMatrix(S)
        plan = dm.plan(8)
        th = np.ones(4)
        with pytest.raises(ValueError, match="col0"):
            plan.run(th, 1, omega_kind=1, col0=1, d_global=16)
        with pytest.raises(ValueError):
            plan.run(th, 1, omega_kind=1, col0=0, d_global=4)
        with pytest.raises(ValueError, match="finite"):
            plan.run(np.array([1.0, np.nan]), 1, omega_kind=1)
        with pytest.raises(ValueError):
            plan.run(th, 0, omega_kind=1)
        with pytest.raises(ValueError):
            plan.run(th, 1, omega_kind=0)  # GIVEN without a block
        with pytest.raises(ValueError, match="begin"):
            plan.step(1)
        with pytest.raises(ValueError):
            plan.set_option(_lib.OPT_E_FOLD, 7)
        with pytest.raises(ValueError):
            plan.set_option(99, 1)
        with pytest.raises(ValueError):
            dm.scale(0.0)
        dm.close()

    def test_matrix_checks(self):
        S = graphs.sbm(200, 2, 5.0, 1.0, seed=2)
        bad = pb.SparseMatrix(S.n_rows, 10, S.row_offsets, S.col_indices % 10, S.values, check=False)
        with pytest.raises(ValueError, match="column index"):
            pb.DeviceMatrix(pb.SparseMatrix(S.n_rows, 5, S.row_offsets, S.col_indices, S.values, check=False))
        dm = pb.DeviceMatrix(bad)  # valid columns (mod 10) but a non-square matrix
        with pytest.raises(ValueError, match="square"):
            dm.plan(4).run(np.ones(3), 1, omega_kind=1)
        dm.close()
        sq = pb.DeviceMatrix(S)
        with pytest.raises(ValueError):
            sq.plan(4).partition(0, S.n_rows + 5, 0)
        sq.close()


class TestReferenceSuiteOnDevice:
    """The reference suite's numerical criteria, run through the device path."""

    def test_linearity_in_function(self):  # tests/test_engine.py:132-150
        rng = np.random.default_rng(8)
        n = 40
        a = rng.standard_normal((n, n))
        a = 0.5 * (a + a.T)
        a *= 0.95 / np.linalg.norm(a, 2)
        S = pb.SparseMatrix.from_dense(a)
        om = O.sample_projection(n, 5, 8)
        f, g = pb.indicator_above(0.2), pb.constant(1.0)
        quad = pb.QuadratureSpec(breakpoints=(0.2,))
        combo = lambda x: 0.6 * np.asarray(f(x)) - 1.1 * np.asarray(g(x))  # noqa: E731
        lhs = pb.fast_embed_eig(S, combo, 25, om, quadrature=quad).values
        rhs = 0.6 * pb.fast_embed_eig(S, f, 25, om, quadrature=quad).values - 1.1 * pb.fast_embed_eig(
            S, g, 25, om, quadrature=quad).values
        assert np.linalg.norm(lhs - rhs) <= 1e-12 * max(1.0, np.linalg.norm(rhs))

    def test_a9_norm_estimator_band(self):  # tests/test_acceptance.py:357-386
        rng = np.random.default_rng(99)
        for i in range(50):
            lam = np.concatenate([[1.0 if i % 2 else -1.0], rng.uniform(-0.85, 0.85, 199)])
            q, _ = np.linalg.qr(rng.standard_normal((200, 200)))
            dense = (q * lam) @ q.T
            est = pb.estimate_spectral_norm(pb.SparseMatrix.from_dense(dense), pb.EmbedConfig(L=1, d=1, seed=1000 + i))
            assert 0.99 <= est / np.abs(lam).max() <= 1.01 + 1e-12

    def test_a1_polynomial_exactness(self):  # tests/test_acceptance.py:36-56
        rng = np.random.default_rng(101)
        n = 100
        dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.05)
        dense = 0.5 * (dense + dense.T)
        dense /= np.linalg.norm(dense, 2)
        om = O.sample_projection(n, 16, 11)
        emb = pb.fast_embed_eig(pb.SparseMatrix.from_dense(dense), lambda x: 0.3 + 0.5 * x - 0.2 * x**3, 3, om)
        oracle = 0.3 * om + 0.5 * (dense @ om) - 0.2 * np.linalg.matrix_power(dense, 3) @ om
        assert np.linalg.norm(emb.values - oracle) / np.linalg.norm(oracle) <= 1e-10


def test_fuzz_random_csr_bit_exact():
    """Random CSR shapes (empty rows, heavy rows, odd widths) vs the oracle."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @settings(max_examples=int(os.environ.get("CSEMB_FUZZ_EXAMPLES", "40")), deadline=None)
    @given(n=st.integers(1, 400), density=st.floats(0.0, 0.2), heavy=st.booleans(), d=st.integers(1, 70),
           L=st.integers(0, 9), seed=st.integers(0, 2**31), f32=st.booleans())
    def check(n, density, heavy, d, L, seed, f32):
        rng = np.random.default_rng(seed)
        a = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
        if heavy and n > 2:
            a[n // 2, :] = rng.standard_normal(n)
        a = 0.5 * (a + a.T)
        nrm = np.linalg.norm(a, 2) if a.any() else 1.0
        S = pb.SparseMatrix.from_dense(a / (1.05 * nrm))
        om = O.sample_projection(n, d, seed % 1000)
        th = rng.standard_normal(L + 1) * 0.5
        ref, _, _ = O.run_stage(O.CSR.of(S), th, om)
        dm = pb.device_matrix(S, "float32" if f32 else "float64")
        plan = dm.plan(d)
        plan.set_load_balance(split_threshold=64 if heavy else 4096)
        got = plan.apply(th, 1, om)
        if f32:
            assert rel(got, ref) <= 1e-4 or np.linalg.norm(ref) < 1e-6
        elif heavy and n > 64:
            assert rel(got, ref) <= 1e-13 or np.linalg.norm(ref) == 0
        else:
            assert np.array_equal(got, ref)

    check()


def test_graph_replay_bit_exact(config1):
    """CSEMB_OPT_GRAPH: the 2nd identical run is captured, later ones replay the
    CUDA graph -- every run bit-identical to the reference, a changed signature
    (seed, coefficients) re-captures, events still time the replay."""
    z, meta = config1
    S = sparse_from(z)
    dm = pb.DeviceMatrix(S, "float64")
    plan = dm.plan(40)
    for mode in (1, 0, -1):
        plan.set_option(_lib.OPT_GRAPH, mode)
        for _ in range(4):
            plan.run(z["coeffs"], 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=0)
            assert sha(plan.download()) == meta["E_sha256"]
            tot, steps, launches = plan.timing()
            assert tot > 0 and steps > 0 and launches == 60
    other, _, _ = O.apply_expansion(O.CSR.of(S), z["coeffs"][:31], O.sample_projection(2000, 40, 3))
    plan.set_option(_lib.OPT_GRAPH, 1)
    for _ in range(3):
        plan.run(z["coeffs"][:31], 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=3)
        assert np.array_equal(plan.download(), other)
        plan.run(z["coeffs"], 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=0)
        assert sha(plan.download()) == meta["E_sha256"]
    with pytest.raises(ValueError):
        plan.set_option(_lib.OPT_GRAPH, 2)
    dm.close()


def test_graph_survives_buffer_reallocation(config1):
    """A recorded graph has the diagnostics buffer built in: runs of order
    a, a, b > a, a (the b run reallocates the buffer) must neither replay into
    the freed buffer nor report stale diagnostics."""
    z, meta = config1
    S = sparse_from(z)
    dm = pb.DeviceMatrix(S, "float64")
    plan = dm.plan(40)
    plan.set_option(_lib.OPT_GRAPH, 1)
    plan.set_exact_peaks(True)
    om = O.sample_projection(2000, 40, 0)
    refs = {}
    for L in (4, 4, 4, 9, 4, 4, 9, 9, 4, 15, 4):
        th = z["coeffs"][:L + 1]
        if L not in refs:
            refs[L] = O.run_stage(O.CSR.of(S), th, om)
        ref, ref_peaks, _ = refs[L]
        plan.run(th, 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=0)
        assert np.array_equal(plan.download(), ref), L
        peaks, bad, _ = plan.diagnostics()
        assert bad == 0 and peaks.shape == (1, L, 2)
        assert np.array_equal(peaks[0], ref_peaks), L
    dm.close()


def test_out_of_memory_is_reported_and_context_survives(config1):
    """An impossible allocation surfaces as MemoryError (CSEMB_ERR_NOMEM after
    the pool is trimmed and the allocation retried); the context stays usable."""
    z, meta = config1
    dm = pb.DeviceMatrix(sparse_from(z), "float64")
    with pytest.raises(MemoryError):
        dm.plan(1_000_000_000)  # 3 x 2000 x 1e9 doubles
    plan = dm.plan(40)
    plan.run(z["coeffs"], 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=0)
    assert sha(plan.download()) == meta["E_sha256"]
    dm.close()


def test_repeated_create_destroy_does_not_grow_memory(config1):
    """Matrices and plans come from the context's stream-ordered pool: many
    create / run / destroy cycles reuse blocks instead of growing usage."""
    import torch

    z, meta = config1
    S = sparse_from(z)

    def cycle():
        dm = pb.DeviceMatrix(S, "float64")
        out = dm.plan(40).apply(z["coeffs"], 1, None, omega_kind=_lib.OMEGA_SPLITMIX)
        dm.close()
        return out

    first = cycle()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(25):
        assert np.array_equal(cycle(), first)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, (free0, free1)
    assert sha(first) == meta["E_sha256"]


@pytest.mark.parametrize("kind,n,d,L,row_order", [
    ("sbm", 200_000, 80, 6, -1),        # windowed batch-count buckets (auto)
    ("sbm", 150_000, 24, 7, 2),         # windowed, narrow rows (G = 4)
    ("chung_lu", 200_000, 40, 6, -1),   # skewed: global buckets (auto)
    ("chung_lu", 120_000, 130, 5, 4096),  # explicit window, column tiling
    ("random", 150_000, 8, 6, 1),       # global buckets on a uniform graph
])
def test_schedule_orders_bit_exact_at_scale(kind, n, d, L, row_order):
    """Medium-scale bit-exactness of the fused recurrence under every row
    schedule (windowed / global batch-count buckets, natural), f64, against
    the C oracle.  Row splitting off so every row keeps stored order."""
    if kind == "sbm":
        S = graphs.sbm(n, 20, 12.0, 4.0, seed=n)
    elif kind == "chung_lu":
        S = graphs.chung_lu(n, seed=3)
    else:
        rng = np.random.default_rng(n)
        S = pb.normalized_adjacency(rng.integers(0, n, size=(8 * n, 2)), n)
    th = pb.legendre_coefficients(pb.indicator_above(0.6), L).coeffs
    om = O.sample_projection(n, d, 5)
    ref = _oracle_embed(S, th, om)
    dm = pb.DeviceMatrix(S, "float64")
    plan = dm.plan(d)
    plan.set_load_balance(split_threshold=0, row_order=row_order)
    got = plan.apply(th, 1, om)
    assert np.array_equal(got, ref)
    plan.set_load_balance(row_order=0)
    assert np.array_equal(plan.apply(th, 1, om), ref)
    dm.close()


# --------------------------------------------------------------------------
# BASELINE sizes: config 2 in full against the oracle; configs 3 / 4 in full
# through the fp32 gates against the (bit-exact) fp64 device result
# --------------------------------------------------------------------------
def _device_result(plan, d):
    """E of the plan's last run as an (n, d) torch tensor (device to device)."""
    import torch

    ptr, ld, dt = plan.output()
    out = torch.empty((plan.dm.n_rows, d), dtype=torch.float64 if dt == 0 else torch.float32, device="cuda")
    plan.copy_output_to(out.data_ptr(), d)
    plan.dm.ctx.sync()
    return out


def _fp32_gates(E32, E64, n, seed):
    """north_star fp32 gates on device tensors: relative Frobenius error and the
    row-normalised cosine error on 10^4 sampled row pairs."""
    import torch

    a, b = E32.double(), E64
    r = float(torch.linalg.norm(a - b) / torch.linalg.norm(b))
    pairs = torch.from_numpy(O.sample_pairs(n, 10_000, seed)).cuda()

    def cos(X):
        u, v = X[pairs[:, 0]], X[pairs[:, 1]]
        den = torch.linalg.norm(u, dim=1) * torch.linalg.norm(v, dim=1)
        return torch.where(den > 0, (u * v).sum(1) / den, torch.zeros_like(den))

    return r, float((cos(a) - cos(b)).abs().max())


def test_config2_full_scale_fp64_bit_exact_and_fp32_gates():
    # BASELINE configs[1] at its full size and order: SBM n=1e6 (100 blocks,
    # degree 15 intra + 5 inter), d=80, L=180, f=1{x>=0.95}, the reference's
    # SplitMix projection (seed 0).  fp64 against the oracle, bit for bit
    # (~30 s of 16-thread CPU); fp32 through the north_star gates.
    n, d, L = 1_000_000, 80, 180
    S = graphs.sbm(n, 100, 15.0, 5.0, seed=2)
    th = pb.legendre_coefficients(pb.indicator_above(0.95), L).coeffs
    p64 = pb.DeviceMatrix(S).plan(d)
    p64.run(th, 1, omega_kind=1, seed=0)
    E64 = _device_result(p64, d)
    ref, _, bad = O.run_stage(O.CSR.of(S), th, O.sample_projection(n, d, 0))
    assert bad == 0
    assert np.array_equal(E64.cpu().numpy(), ref)
    del ref
    p32 = pb.DeviceMatrix(S, "float32").plan(d)
    p32.run(th, 1, omega_kind=1, seed=0)
    r, c = _fp32_gates(_device_result(p32, d), E64, n, 3)
    print(f"config 2 full scale: fp64 bit-exact vs oracle; fp32 rel {r:.3e}, cosine error {c:.3e}")
    assert r <= FP32_REL and c <= COS_TOL, (r, c)


# configs 3 / 4 / 5 at full shape against the oracle: tests/test_gpu_scale.py


# --------------------------------------------------------------------------
# value-free normalized adjacency (CSEMB_OPT_VALUE_FREE): K1 recomputes
# 1/sqrt(deg u * deg v) (sparse.py:224) from the row offsets
# --------------------------------------------------------------------------
def _value_free_on(plan) -> bool:
    """Request K1's value-free path.  The shipped build compiles it out (K1_VF=0:
    measured slower, profiles/r2_k1_experiments.txt) and must say so with
    CSEMB_ERR_UNSUPPORTED (NotImplementedError) rather than ignore the request;
    a K1_VF=1 build turns it on (that build passed the whole GPU suite with it
    on by default, round 2)."""
    try:
        plan.set_option(_lib.OPT_VALUE_FREE, 1)
        return True
    except NotImplementedError as e:
        assert "compiled out" in str(e)
        return False


class TestValueFree:
    def test_detected_on_normalized_adjacency_and_bit_exact(self, config1):
        z, meta = config1
        S = sparse_from(z)
        th = pb.legendre_coefficients(pb.indicator_above(0.9), 60).coeffs
        om = O.sample_projection(2000, 40, 0)
        for dt in ("float64", "float32"):
            dm = pb.DeviceMatrix(S, dt)
            assert dm.value_free
            plan = dm.plan(40)
            vf = _value_free_on(plan)
            on = plan.apply(th, 1, om)
            plan.set_option(_lib.OPT_VALUE_FREE, 0)
            off = plan.apply(th, 1, om)
            assert np.array_equal(on, off), f"value-free {'on' if vf else 'compiled out'}"
            if dt == "float64":
                assert sha(on) == meta["E_sha256"]
            dm.close()

    def test_not_detected_on_other_values(self, config1):
        z, _ = config1
        S = sparse_from(z)
        vals = np.asarray(S.values).copy()
        vals[len(vals) // 2] = np.nextafter(vals[len(vals) // 2], 1.0)  # one ulp off the formula
        T = pb.SparseMatrix(S.n_rows, S.n_cols, S.row_offsets, S.col_indices, vals)
        dm = pb.DeviceMatrix(T, "float64")
        assert not dm.value_free
        th = pb.legendre_coefficients(pb.indicator_above(0.9), 20).coeffs
        om = O.sample_projection(2000, 40, 0)
        plan = dm.plan(40)
        _value_free_on(plan)  # requested, but the check says no: values are read
        assert np.array_equal(plan.apply(th, 1, om), _oracle_embed(T, th, om))
        dm.close()

    def test_scale_clears_it(self, config1):
        z, _ = config1
        S = sparse_from(z)
        dm = pb.DeviceMatrix(S, "float64")
        plan = dm.plan(40)
        th = pb.legendre_coefficients(pb.indicator_above(0.9), 12).coeffs
        om = O.sample_projection(2000, 40, 0)
        plan.apply(th, 1, om)  # the check ran and cached "on"
        assert dm.value_free
        dm.scale(0.5)
        assert not dm.value_free
        T = pb.SparseMatrix(S.n_rows, S.n_cols, S.row_offsets, S.col_indices, np.asarray(S.values) * 0.5)
        assert np.array_equal(plan.apply(th, 1, om), _oracle_embed(T, th, om))
        dm.close()

    def test_config2_full_size_on_off_identical(self):
        # BASELINE config 2's graph: both dtypes, value-free on vs off bit-identical
        # (heavy-row chunks none here; row order windows as in the bench)
        S = graphs.sbm(1_000_000, 100, 15.0, 5.0, seed=2)
        th = pb.legendre_coefficients(pb.indicator_above(0.95), 8).coeffs
        for dt in ("float64", "float32"):
            dm = pb.DeviceMatrix(S, dt)
            assert dm.value_free
            plan = dm.plan(80)
            if not _value_free_on(plan):
                dm.close()
                continue  # compiled out: nothing to compare at this size
            plan.run(th, 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=7)
            a = _device_result(plan, 80)
            plan.set_option(_lib.OPT_VALUE_FREE, 0)
            plan.run(th, 1, omega_kind=_lib.OMEGA_SPLITMIX, seed=7)
            b = _device_result(plan, 80)
            assert bool((a == b).all())
            dm.close()


def test_fuzz_split_exchange_bit_exact():
    """Random CSR shapes through the split exchange (csemb_plan_partition_split)
    with 1-4 emulated ranks: fp64 bit-identical to the split-order restatement
    (strict stored order inside each part), within rounding of the 1-GPU order."""
    import torch
    from hypothesis import given, settings
    from hypothesis import strategies as st

    from conftest import split_order_stage
    from paper_1509_08360_b200.distributed import local_rows, row_blocks

    @settings(max_examples=int(os.environ.get("CSEMB_FUZZ_EXAMPLES", "25")), deadline=None)
    @given(n=st.integers(1, 300), density=st.floats(0.0, 0.2), d=st.integers(1, 40), L=st.integers(1, 7),
           world=st.integers(1, 4), seed=st.integers(0, 2**31))
    def check(n, density, d, L, world, seed):
        rng = np.random.default_rng(seed)
        a = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
        a = 0.5 * (a + a.T)
        nrm = np.linalg.norm(a, 2) if a.any() else 1.0
        S = pb.SparseMatrix.from_dense(a / (1.05 * nrm))
        th = rng.standard_normal(L + 1) * 0.5
        om = O.sample_projection(n, d, seed % 1000)
        n_pad, blocks = row_blocks(n, world)
        ld = -(-d // 2) * 2
        F = torch.zeros((world * n_pad, ld), dtype=torch.float64, device="cuda")
        ranks = []
        for lo, hi in blocks:
            if hi <= lo:
                continue
            dm = pb.DeviceMatrix(local_rows(S, lo, hi), "float64")
            plan = dm.plan(d)
            plan.set_load_balance(split_threshold=0)
            q = [torch.zeros((n_pad, ld), dtype=torch.float64, device="cuda") for _ in range(2)]
            plan.partition_split(lo, n, F.data_ptr(), q[0].data_ptr(), q[1].data_ptr())
            torch.cuda.synchronize()
            plan.begin(th, omega_kind=1, seed=seed % 1000)
            ranks.append((lo, hi, dm, plan, q))
        for _, _, dm, _, _ in ranks:
            dm.ctx.sync()
        for r in range(1, L + 1):
            for *_, plan, _ in ranks:
                plan.step_local(r)
            for *_, plan, _ in ranks:
                plan.step(r)
            for _, _, dm, _, _ in ranks:
                dm.ctx.sync()
            if r < L:
                for lo, hi, dm, plan, q in ranks:
                    F[lo:hi] = q[r & 1][:hi - lo]
                torch.cuda.synchronize()
        got = []
        for lo, hi, dm, plan, q in ranks:
            plan.end(False)
            got.append(plan.download())
            dm.close()
        got = np.concatenate(got)
        assert np.array_equal(got, split_order_stage(O.CSR.of(S), th, om, blocks))
        ref, _, _ = O.run_stage(O.CSR.of(S), th, om)
        assert rel(got, ref) <= 1e-12 or np.linalg.norm(ref) < 1e-300

    check()
