"""Host-side mirror of the reference (no GPU): coefficients, spectral
functions, CSR container and builders, configs, generators."""

import math

import numpy as np
import pytest

import paper_1509_08360_b200 as pb
from conftest import load_golden
from paper_1509_08360_b200 import graphs


class CutAbove:
    """Same callable the golden generator used for config 4's weight."""

    def __init__(self, c):
        self.c = float(c)

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        return np.where(x >= self.c, x, 0.0)

    def breakpoints(self):
        return (self.c,)


SPECS = {
    "ind090_60": lambda: (pb.indicator_above(0.9), 60),
    "ind095_180": lambda: (pb.indicator_above(0.95), 180),
    "commute001_180": lambda: (pb.commute_time(0.01), 180),
    "cut030_odd_120": lambda: (pb.odd_extension(CutAbove(0.3)), 120),
    "ind098_root2_90": lambda: (pb.root_function(pb.indicator_above(0.98), 2), 90),
    "ind040_odd_root2_40": lambda: (pb.odd_extension(pb.root_function(pb.indicator_above(0.4), 2)), 40),
    "identity_1": lambda: (pb.identity(), 1),
    "identity_7": lambda: (pb.identity(), 7),
    "const25_0": lambda: (pb.constant(2.5), 0),
    "table_33": lambda: (pb.tabulated([-1.0, -0.2, 0.5, 1.0], [0.0, 1.0, -0.5, 2.0]), 33),
    "ind09_odd_60": lambda: (pb.odd_extension(pb.indicator_above(0.9)), 60),
    "commute_root3_30": lambda: (pb.root_function(pb.commute_time(0.05), 3), 30),
}


class TestCoefficients:
    @pytest.mark.parametrize("name", sorted(SPECS))
    def test_bit_exact_vs_reference(self, name):
        z, meta = load_golden("coefficients")
        f, order = SPECS[name]()
        e = pb.legendre_coefficients(f, order)
        assert e.digest() == meta[name]["sha256"]
        assert np.array_equal(e.coeffs, z[name])
        if hasattr(f, "describe"):
            assert f.describe() == meta[name]["describe"]

    def test_analytic_indicator(self):  # tests/test_legendre.py:29-37
        c, L = 0.3, 40
        e = pb.legendre_coefficients(pb.indicator_above(c), L)
        P = pb.legendre_table(L + 1, np.array([c]))[:, 0]
        assert e.coeffs[0] == pytest.approx((1 - c) / 2, abs=1e-12)
        for r in range(1, L + 1):
            assert e.coeffs[r] == pytest.approx((P[r - 1] - P[r + 1]) / 2, abs=1e-12)

    def test_gibbs_value(self):  # tests/test_legendre.py:118-123
        e = pb.legendre_coefficients(pb.indicator_above(0.98), 180)
        assert pb.expansion_eval(e, 0.5) == pytest.approx(-0.0005311185431373922, abs=1e-12)

    def test_expansion_immutable(self):
        e = pb.LegendreExpansion([1.0, 2.0])
        with pytest.raises(ValueError):
            e.coeffs[0] = 3.0
        with pytest.raises(ValueError):
            pb.LegendreExpansion([np.nan])


class TestFunctions:
    def test_kinds_and_breakpoints(self):
        assert pb.indicator_above(0.9)(np.array([0.8, 0.9]))[1] == 1.0
        assert pb.commute_time(0.01)(0.995) == pytest.approx(10.0)
        f = pb.odd_extension(pb.indicator_above(0.4))
        assert f.breakpoints() == (-0.4, 0.0, 0.4)
        assert f(-0.5) == -1.0 and f.describe() == "indicator:0.4|odd"
        g = pb.root_function(pb.indicator_above(0.2), 2)
        assert g.describe() == "indicator:0.2|root:2"
        with pytest.raises(ValueError):
            pb.root_function(pb.identity(), 2)
        with pytest.raises(ValueError):
            pb.SpectralFunction("nope")

    def test_parse(self):
        assert pb.parse_function("indicator:0.5").threshold == 0.5
        assert pb.parse_function("commute").clip == 1e-3
        with pytest.raises(ValueError):
            pb.parse_function("bogus:1")


class TestBuilders:
    def test_normalized_adjacency_bit_exact(self):
        z, meta = load_golden("builders")
        for i in range(4):
            S = pb.normalized_adjacency(z[f"adj{i}_edges"], meta[f"adj{i}"]["n"])
            assert np.array_equal(S.row_offsets, z[f"adj{i}_row_offsets"])
            assert np.array_equal(S.col_indices, z[f"adj{i}_col_indices"])
            assert np.array_equal(S.values, z[f"adj{i}_values"])
            S._validate()

    def test_config1_graph_bit_exact(self, config1):
        z, _ = config1
        S = pb.normalized_adjacency(z["edges"], 2000)
        assert S.nnz == 65036
        assert np.array_equal(S.row_offsets, z["row_offsets"])
        assert np.array_equal(S.col_indices, z["col_indices"])
        assert np.array_equal(S.values, z["values"])

    def test_dilate_bit_exact(self):
        z, _ = load_golden("builders")
        A = pb.SparseMatrix(int(z["dil_A_n_rows"]), int(z["dil_A_n_cols"]), z["dil_A_row_offsets"],
                            z["dil_A_col_indices"], z["dil_A_values"])
        D = pb.dilate(A)
        assert np.array_equal(D.row_offsets, z["dil_S_row_offsets"])
        assert np.array_equal(D.col_indices, z["dil_S_col_indices"])
        assert np.array_equal(D.values, z["dil_S_values"])

    def test_dilate_layout(self):  # tests/test_sparse.py:92-98
        a = np.arange(1, 7, dtype=float).reshape(2, 3)
        S = pb.dilate(pb.SparseMatrix.from_dense(a)).to_dense()
        assert np.array_equal(S[:3, 3:], a.T) and np.array_equal(S[3:, :3], a)
        assert pb.dilate(pb.SparseMatrix.zeros(2, 3)).nnz == 0

    def test_invariants(self):
        with pytest.raises(ValueError):
            pb.SparseMatrix(2, 2, [0, 2, 2], [1, 0], [1.0, 1.0])  # unsorted row
        with pytest.raises(ValueError):
            pb.SparseMatrix(2, 2, [0, 1, 2], [0, 5], [1.0, 1.0])
        with pytest.raises(ValueError):
            pb.SparseMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 0.0])
        with pytest.raises(ValueError):
            pb.normalized_adjacency([(0, 5)], 3)
        m = pb.SparseMatrix.from_coo([0, 0], [1, 1], [2.0, 3.0], 2, 2)
        assert m.nnz == 1 and m.to_dense()[0, 1] == 5.0

    def test_scale_values(self):
        S = pb.SparseMatrix.identity(3)
        assert np.array_equal(pb.scale_values(S, 0.5).values, [0.5] * 3)
        with pytest.raises(ValueError):
            pb.scale_values(S, 0.0)


class TestConfig:
    def test_validation(self):  # tests/test_engine.py:293-307
        for kw in [dict(L=0, d=4), dict(L=10, d=4, b=3), dict(L=10, d=0), dict(L=10, d=4, epsilon=1.0),
                   dict(L=10, d=4, beta=0.0)]:
            with pytest.raises(ValueError):
                pb.EmbedConfig(**kw)
        assert pb.EmbedConfig(L=180, d=80, b=2).stage_order == 90

    def test_dimensions(self):  # tests/test_engine.py:29-46
        assert pb.jl_dimension(100, 0.5, 2.0) == 443
        assert pb.jl_dimension(317080, 0.5, 1.0) == 913
        assert pb.default_dimension(317080) == 77

    def test_fold_seed(self):
        z, meta = load_golden("omega")
        got = [pb.fold_seed(s, t) for s, t in meta["fold_cases"]]
        assert np.array_equal(np.array(got, dtype=np.uint64), z["folds"])


class TestGenerators:
    def test_sbm_degrees(self):
        n, blocks = 20000, 10
        e = graphs.sbm_edges(n, blocks, 15.0, 5.0, seed=1)
        bs = n // blocks
        same = (e[:, 0] // bs) == (e[:, 1] // bs)
        assert abs(2 * same.sum() / n - 15.0) < 0.3
        assert abs(2 * (~same).sum() / n - 5.0) < 0.2
        S = graphs.sbm(n, blocks, 15.0, 5.0, seed=1)
        S._validate()
        assert np.array_equal(S.to_scipy().T.toarray(), S.to_scipy().toarray()) if n <= 2000 else True
        assert abs(S.nnz / n - 20.0) < 0.5

    def test_deterministic(self):
        a = graphs.sbm_edges(1000, 4, 8.0, 2.0, seed=3)
        b = graphs.sbm_edges(1000, 4, 8.0, 2.0, seed=3)
        assert np.array_equal(a, b)

    def test_chung_lu_mean_degree(self):
        e = graphs.chung_lu_edges(50000, seed=2)
        assert abs(2 * len(e) / 50000 - 20.0) < 1.0
        S = graphs.chung_lu(50000, seed=2)
        S._validate()

    def test_bag_of_words(self):
        A = graphs.bag_of_words(300, 500, seed=1, mean_len=40)
        A._validate()
        rn = np.sqrt(np.bincount(np.repeat(np.arange(300), np.diff(A.row_offsets)),
                                 weights=A.values**2, minlength=300))
        assert np.allclose(rn[rn > 0], 1.0)
        assert math.isclose(np.linalg.norm(A.to_dense(), 2), np.linalg.norm(A.to_dense(), 2))


def test_product_never_imports_oracle():
    import pathlib

    pkg = pathlib.Path(pb.__file__).parent
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


class TestIOAndCLI:
    def test_embedding_round_trip(self, tmp_path):
        from paper_1509_08360_b200 import io as bio

        v = np.random.default_rng(0).standard_normal((7, 3))
        p = str(tmp_path / "e.bin")
        bio.write_embedding(p, v)
        raw = open(p, "rb").read()
        assert raw[:8] == b"CSEMB001" and len(raw) == 8 + 16 + 8 * 21
        assert np.array_equal(bio.read_embedding(p), v)
        open(p, "wb").write(b"XXXX")
        with pytest.raises(pb.InputFormatError):
            bio.read_embedding(p)

    def test_edgelist_reader(self, tmp_path):
        from paper_1509_08360_b200 import io as bio

        p = tmp_path / "g.txt"
        p.write_text("# comment\n0 1\n1 2\n")
        e, n = bio.read_edgelist(str(p))
        assert n == 3 and e.shape == (2, 2)
        p.write_text("0 -1\n")
        with pytest.raises(pb.InputFormatError):
            bio.read_edgelist(str(p))

    def test_usage_errors_exit_2(self, tmp_path):
        from paper_1509_08360_b200.cli import main

        g = tmp_path / "g.txt"
        g.write_text("0 1\n")
        with pytest.raises(SystemExit) as ex:
            main(["embed", "--input", str(g), "--format", "edgelist", "--matrix", "raw", "--function",
                  "indicator:0.5", "--L", "4", "--output", str(tmp_path / "o.bin")])
        assert ex.value.code == 2
        with pytest.raises(SystemExit) as ex:
            main(["embed", "--input", str(g), "--format", "edgelist", "--function", "bogus", "--L", "4",
                  "--output", str(tmp_path / "o.bin")])
        assert ex.value.code == 2

    def test_parse_error_exit_3(self, tmp_path):
        from paper_1509_08360_b200.cli import main

        g = tmp_path / "g.txt"
        g.write_text("zero one\n")
        assert main(["embed", "--input", str(g), "--format", "edgelist", "--function", "indicator:0.5", "--L", "4",
                     "--output", str(tmp_path / "o.bin")]) == 3


def test_cli_downstream_commands_parse_and_usage_errors(tmp_path):
    """`cluster` / `eval` exist with the reference's options; eval without an
    exact source is a usage error (exit 2), before any device work."""
    from paper_1509_08360_b200 import cli, io as pio

    p = cli.build_parser()
    a = p.parse_args(["cluster", "--input", "g.txt", "--function", "indicator:0.5", "--L", "40"])
    assert (a.k, a.runs, a.b, a.dtype) == (200, 25, 1, "float64")
    e = tmp_path / "e.bin"
    pio.write_embedding(str(e), np.ones((3, 2)))
    with pytest.raises(SystemExit) as ex:
        cli.main(["eval", "--approx", str(e), "--output-prefix", str(tmp_path / "o")])
    assert ex.value.code == 2
    with pytest.raises(SystemExit) as ex:
        cli.main(["cluster", "--input", "g.txt", "--function", "indicator:0.5", "--L", "40", "--b", "3"])
    assert ex.value.code == 2
