"""Pin the CPU oracle against the reference's golden vectors (no GPU).

The fixtures in tests/golden/ were produced by running the reference itself
(tests/golden/make_golden.py); these tests prove the oracle restates it
bit-for-bit before any device result is checked against the oracle.
"""

import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import csr_from, load_golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class TestOmega:
    def test_golden_signs(self):
        z, meta = load_golden("omega")
        for n, d, seed in meta["cases"]:
            om = O.sample_projection(n, d, seed)
            assert np.array_equal(np.packbits(om > 0), z[f"signs_{n}_{d}_{seed}"])
            assert np.all(np.abs(om) == 1.0 / np.sqrt(d))

    def test_frozen_pattern(self):  # tests/test_engine.py:60-65
        om = O.sample_projection(3, 4, 42) * 2.0
        assert np.array_equal(om, [[-1, 1, -1, 1], [-1, 1, 1, -1], [1, 1, 1, 1]])

    def test_numpy_restatement_agrees(self):
        for n, d, s in [(50, 9, 3), (37, 80, 2**63 + 11)]:
            assert np.array_equal(O.sample_projection(n, d, s), O.np_sample_projection(n, d, s))

    def test_column_slice_uses_global_d(self):
        full = O.sample_projection(40, 80, 5)
        assert np.array_equal(O.sample_projection(40, 80, 5, col0=24, w=13), full[:, 24:37])

    def test_fold_seed(self):
        z, meta = load_golden("omega")
        got = [O.fold_seed(s, t) for s, t in meta["fold_cases"]]
        assert np.array_equal(np.array(got, dtype=np.uint64), z["folds"])


class TestRecurrence:
    def test_config1_bit_exact(self, config1):
        z, meta = config1
        S = csr_from(z)
        E, peaks, bad = O.run_stage(S, z["coeffs"], O.sample_projection(2000, 40, 0))
        assert bad == 0
        assert sha(E) == meta["E_sha256"]
        assert np.array_equal(E, z["E"])

    def test_config1_step_log(self, config1):
        z, _ = config1
        _, peaks, _ = O.run_stage(csr_from(z), z["coeffs"], O.sample_projection(2000, 40, 0))
        ref = z["step_max_abs"]  # (r, col0, max_abs) from the reference's debug log (%.6e)
        got = peaks[ref[:, 0].astype(int) - 1, ref[:, 1].astype(int) // 32]
        np.testing.assert_allclose(got, ref[:, 2], rtol=5e-7)

    def test_cascade_two_stages(self, small_cases):
        z, _ = small_cases
        out, bad, _ = O.apply_expansion(csr_from(z, "cascade_"), _stage_coeffs("ind098_root2_90"),
                                        O.sample_projection(80, 8, 13), n_stages=2)
        assert bad == 0 and np.array_equal(out, z["cascade_E"])

    def test_general_dilation(self, small_cases):
        z, _ = small_cases
        S = O.CSR(420, 420, z["general2_dilated_row_offsets"], z["general2_dilated_col_indices"],
                  z["general2_dilated_values"])
        out, _, _ = O.run_stage(S, _stage_coeffs("cut030_odd_120"), O.sample_projection(420, 24, 4))
        assert np.array_equal(out[120:], z["general2_rows"])
        assert np.array_equal(out[:120], z["general2_cols"])

    def test_chunk_crossing_width(self, small_cases):
        z, _ = small_cases
        S = csr_from(z, "wide_")
        from paper_1509_08360_b200 import indicator_above, legendre_coefficients

        th = legendre_coefficients(indicator_above(0.0), 12).coeffs
        out, peaks, _ = O.run_stage(S, th, O.sample_projection(50, 70, 10))
        assert np.array_equal(out, z["wide_E"])
        ref = z["wide_steps"]
        np.testing.assert_allclose(peaks[ref[:, 0].astype(int) - 1, ref[:, 1].astype(int) // 32],
                                   ref[:, 2], rtol=5e-7)

    def test_polynomial_case(self, small_cases):
        z, _ = small_cases
        out, _, _ = O.run_stage(csr_from(z, "poly_"), z["poly_theta"], O.sample_projection(150, 10, 0))
        assert np.array_equal(out, z["poly_E"])

    def test_divergence_first_bad_r(self, small_cases):
        _, meta = small_cases
        S = O.CSR(4, 4, np.arange(5), np.arange(4), np.full(4, 10.0))
        th = np.zeros(251)
        th[1] = 1.0  # identity() expansion
        _, _, bad = O.run_stage(S, th, O.sample_projection(4, 2, 0))
        assert bad == meta["divergence"]["first_bad_r"] == 239

    def test_thread_count_invariance(self, config1):
        z, _ = config1
        S = csr_from(z)
        om = O.sample_projection(2000, 40, 0)
        O.set_threads(1)
        a, _, _ = O.run_stage(S, z["coeffs"][:8], om)
        O.set_threads(max(2, O.num_threads()))
        b, _, _ = O.run_stage(S, z["coeffs"][:8], om)
        assert np.array_equal(a, b)


def _stage_coeffs(name):
    z, _ = load_golden("coefficients")
    return z[name]


class TestSpmm:
    def test_kats(self):  # tests/test_sparse.py:52-79
        S = O.CSR(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0])
        assert np.array_equal(O.spmm(S, np.array([[1.0], [2.0]])), [[2.0], [1.0]])
        Z = O.CSR(3, 4, [0, 0, 0, 0], [], [])
        assert np.array_equal(O.spmm(Z, np.ones((4, 2))), np.zeros((3, 2)))

    def test_matches_scipy_order(self, config1):
        import scipy.sparse as sp

        z, _ = config1
        S = csr_from(z)
        X = np.random.default_rng(0).standard_normal((2000, 7))
        ref = sp.csr_array((S.values, S.col_indices, S.row_offsets), shape=(2000, 2000)) @ X
        assert np.array_equal(O.spmm(S, X), ref)


class TestNormAndPairs:
    def test_spectral_norm_golden(self):
        z, meta = load_golden("norm")
        for name, m in meta.items():
            S = csr_from(z, name + "_")
            est = O.spectral_norm(S, m["seed"], m["norm_iters"], m["norm_vectors_factor"], m["norm_safety"])
            assert est == pytest.approx(m["estimate"], rel=1e-12, abs=1e-15)

    def test_pairs_golden(self, config1):
        z, _ = config1
        assert np.array_equal(O.sample_pairs(2000, 10_000, 0), z["pairs"])

    def test_row_normalize_zero_rows(self):
        E = np.array([[3.0, 4.0], [0.0, 0.0]])
        assert np.array_equal(O.row_normalize(E), [[0.6, 0.8], [0.0, 0.0]])
        c = O.pair_cosines(E, np.array([[0, 1]]))
        assert c[0] == 0.0
