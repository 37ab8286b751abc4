"""Downstream consumers on the device vs the reference's
fixtures and the oracle (B200 only).

Bars: labels, iteration counts and modularity identical to the reference;
inertia histories within 1e-10 relative (the reference's X @ C.T comes from
BLAS in unspecified order; ours follows numpy's pairwise order); centroids
bit-identical to np.add.at means of the same labels; pair cosines within
1e-12; distortion percentiles within 1e-10.
"""

import numpy as np
import pytest

import oracle as O
import paper_1509_08360_b200 as pb
from conftest import load_golden, sparse_from
from paper_1509_08360_b200 import cluster as pcl
from paper_1509_08360_b200 import distortion as D

pytestmark = pytest.mark.gpu

HIST_REL = 1e-10
COS_ABS = 1e-12


@pytest.fixture(autouse=True)
def _lib_ready(gpu_lib):
    yield


@pytest.fixture(scope="module")
def ds():
    return load_golden("downstream")


@pytest.fixture(scope="module")
def rows(ds, config1):
    z, _ = ds
    c1, _ = config1
    return {"config1": c1["E"], "blobs": z["blobs_X"], "dup": z["dup_X"]}


def _means(X, labels, K):
    acc = np.zeros((K, X.shape[1]))
    np.add.at(acc, labels, X)
    return acc / np.bincount(labels, minlength=K)[:, None]


def _close_hist(got, want, X=None):
    """Inertia histories: 1e-10 relative, plus (given the rows X) the absolute
    cancellation bound of d2 = |x|^2 + |c|^2 - 2 x.c, 16 eps sum |x|^2 -- the
    reference's BLAS X @ C.T leaves a few-ulp residue where ours is exactly 0
    (identical rows)."""
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    atol = 1e-300 if X is None else 16 * np.finfo(np.float64).eps * float(np.sum(np.asarray(X) ** 2))
    assert np.all(np.abs(got - want) <= HIST_REL * np.abs(want) + atol), (got, want)


class TestKMeans:
    def test_reference_fixtures(self, ds, rows):
        z, meta = ds
        for key, m in meta["kmeans"].items():
            a = pcl.kmeans(rows[m["input"]], m["K"], seed=m["seed"])
            assert np.array_equal(a.labels, z[f"km_{key}_labels"]), key
            assert a.n_iters == m["n_iters"], key
            _close_hist(a.inertia_history, z[f"km_{key}_history"])

    def test_duplicate_points_exact_zero_distances(self, ds, rows):
        """Identical rows have distance exactly 0 (pairwise-order dots): the
        zero-total seeding branch and the reseed argmax follow the reference."""
        z, meta = ds
        a = pcl.kmeans(rows["dup"], 8, seed=4)
        assert a.inertia == 0.0 and set(a.inertia_history) == {0.0}
        assert np.array_equal(a.labels, z["km_dup_K8_s4_labels"])

    def test_centroids_bit_identical_to_add_at_means(self, rows):
        X = rows["blobs"]
        km = pcl.DeviceKMeans(X, 3)
        try:
            a = pcl.kmeans(X, 3, seed=2, handle=km)
            assert a.n_iters < 100  # converged: centroids are the means of the final labels
            assert np.array_equal(km.centroids(), _means(X, a.labels, 3))
        finally:
            km.close()

    @pytest.mark.parametrize("n,d,K,seed", [
        (3000, 80, 200, 1),   # centroids staged per 32-wide tile (no CFULL)
        (2500, 150, 6, 2),    # d > 128: several pairwise leaves (k_km_assign_wide)
        (1500, 3, 5, 3),      # d < 8: sequential pairwise leaf
        (4000, 129, 9, 4),    # first d with a split
        (777, 17, 64, 5),     # ragged tiles
    ])
    def test_against_oracle(self, n, d, K, seed):
        rng = np.random.default_rng(seed)
        centers = rng.standard_normal((K, d)) * 3.0
        X = centers[rng.integers(0, K, size=n)] + rng.standard_normal((n, d))
        a = pcl.kmeans(X, K, seed=seed)
        labels, hist = O.kmeans(X, K, seed=seed)
        assert np.array_equal(a.labels, labels)
        _close_hist(a.inertia_history, hist)

    def test_device_rows_and_f32(self, config1):
        """K-means straight from a plan's device-resident E (fp64 and fp32)."""
        c1, _ = config1
        S = sparse_from(c1)
        for dtype in ("float64", "float32"):
            dm = pb.DeviceMatrix(S, dtype)
            plan = dm.plan(40)
            plan.run(c1["coeffs"], 1, omega_kind=pb._lib.OMEGA_SPLITMIX, seed=0)
            E = plan.download()
            a = pcl.kmeans(pcl.plan_rows(plan), 4, seed=0x6B6D6531)
            b = pcl.kmeans(E, 4, seed=0x6B6D6531)
            assert np.array_equal(a.labels, b.labels) and a.inertia_history == b.inertia_history
            dm.close()

    def test_deterministic_and_errors(self, rows):
        X = rows["config1"]
        a, b = pcl.kmeans(X, 9, seed=7), pcl.kmeans(X, 9, seed=7)
        assert np.array_equal(a.labels, b.labels) and a.inertia_history == b.inertia_history
        for K in (0, len(X) + 1):
            with pytest.raises(ValueError):
                pcl.kmeans(X, K)

    def test_single_row_and_k_equals_n(self):
        X = np.arange(12, dtype=np.float64).reshape(4, 3)
        for K in (1, 4):
            a = pcl.kmeans(X, K, seed=1)
            labels, hist = O.kmeans(X, K, seed=1)
            assert np.array_equal(a.labels, labels)
            _close_hist(a.inertia_history, hist)
        a = pcl.kmeans(X[:1], 1)
        assert a.labels.tolist() == [0] and a.inertia == 0.0


class TestModularity:
    def test_reference_fixtures(self, ds, config1):
        z, meta = ds
        c1, _ = config1
        q = pcl.modularity(c1["edges"], c1["labels"])
        assert (q.Q, q.m_edges) == (meta["modularity"]["truth"]["Q"], meta["modularity"]["truth"]["m_edges"])
        for key, want in meta["modularity"].items():
            if key != "truth":
                q = pcl.modularity(c1["edges"], z[f"km_{key}_labels"])
                assert q.Q == want["Q"], key

    def test_duplicates_loops_and_errors(self):
        edges = np.array([[0, 1], [1, 0], [1, 2], [2, 2], [2, 3], [3, 0], [0, 1]])
        lab = np.array([0, 0, 1, 1])
        q = pcl.modularity(edges, lab)
        want, m = O.modularity(edges, lab)
        assert q.Q == want and q.m_edges == m == 4
        with pytest.raises(ValueError):
            pcl.modularity(np.array([[1, 1]]), lab)
        with pytest.raises(ValueError):
            pcl.modularity(edges, lab[:3])

    def test_large_random_graph(self):
        n = 200_000
        edges = np.random.default_rng(5).integers(0, n, size=(1_000_000, 2))
        lab = np.random.default_rng(6).integers(0, 37, size=n)
        q = pcl.modularity(edges, lab)
        want, m = O.modularity(edges, lab)
        assert q.Q == want and q.m_edges == m


class TestPairsAndDistortion:
    def test_pair_cosines_vs_reference(self, ds, config1):
        z, _ = ds
        c1, _ = config1
        cos, zero = D.pair_correlations(c1["E"], c1["pairs"].astype(np.int64))
        assert np.max(np.abs(cos - z["pair_cos"])) <= COS_ABS and not zero.any()

    def test_zero_rows_and_f32(self):
        rng = np.random.default_rng(1)
        E = rng.standard_normal((300, 37))
        E[[3, 77]] = 0.0
        pairs = np.array([[3, 5], [5, 77], [3, 77], [1, 2], [0, 299]])
        cos, zero = D.pair_correlations(E, pairs)
        assert zero.tolist() == [True, True, True, False, False]
        assert np.all(cos[:3] == 0.0)
        assert np.max(np.abs(cos - O.pair_cosines(E, pairs))) <= COS_ABS
        c32, _ = D.pair_correlations(E.astype(np.float32), pairs)
        assert np.max(np.abs(c32 - O.pair_cosines(E.astype(np.float32).astype(np.float64), pairs))) <= COS_ABS
        wide = rng.standard_normal((50, 300))
        pw = D.sample_pairs(50, 200, 0)
        assert np.max(np.abs(D.pair_correlations(wide, pw)[0] - O.pair_cosines(wide, pw))) <= COS_ABS
        with pytest.raises(ValueError):
            D.pair_correlations(E, np.array([[0, 300]]))

    def test_distortion_report_vs_reference(self, ds, config1):
        z, meta = ds
        c1, _ = config1
        for mode in ("deviation", "calibration"):
            rep = D.report_to_dict(D.distortion_percentiles(z["exact_embedding"], c1["E"], n_pairs=20_000, seed=3,
                                                            mode=mode))
            want = meta[f"distortion_{mode}"]
            assert rep["pair_sample_size"] == want["pair_sample_size"]
            assert rep["zero_row_pairs"] == want["zero_row_pairs"]
            if mode == "deviation":
                for k, v in want["percentiles"].items():
                    assert abs(rep["percentiles"][k] - v) <= 1e-10
            else:
                assert [(b["center"], b["count"]) for b in rep["bins"]] == [(b["center"], b["count"])
                                                                            for b in want["bins"]]
                for gb, wb in zip(rep["bins"], want["bins"]):
                    for k, v in wb["percentiles"].items():
                        assert abs(gb["percentiles"][k] - v) <= 1e-10

    def test_device_resident_embedding(self, config1):
        """North-star cosine check without downloading E: fp32 device rows vs
        the fp64 reference on the config-1 pairs (<= 1e-4)."""
        c1, _ = config1
        dm = pb.DeviceMatrix(sparse_from(c1), "float32")
        plan = dm.plan(40)
        plan.run(c1["coeffs"], 1, omega_kind=pb._lib.OMEGA_SPLITMIX, seed=0)
        cos, _ = D.pair_correlations(pcl.plan_rows(plan), c1["pairs"].astype(np.int64))
        assert np.max(np.abs(cos - O.pair_cosines(c1["E"], c1["pairs"]))) <= 1e-4
        dm.close()


def test_cluster_experiment_matches_reference(ds):
    z, meta = ds
    ex_meta = meta["experiment"]
    c1, _ = load_golden("config1")
    ex = pcl.cluster_experiment(c1["edges"].astype(np.int64), 2000, pb.indicator_above(0.9),
                                pb.EmbedConfig(L=60, d=40, seed=0), K=4, runs=5)
    assert list(ex.run_scores) == ex_meta["run_scores"]
    assert ex.median_modularity == ex_meta["median_modularity"]
    assert np.array_equal(ex.median_labels, z["experiment_median_labels"])
    with pytest.raises(ValueError):
        pcl.cluster_experiment(c1["edges"], 2000, pb.indicator_above(0.9), pb.EmbedConfig(L=60, d=40), K=4, runs=0)


def test_modularity_rejects_bad_device_labels(config1):
    """Device-resident labels outside [0, k) are reported, never used as indices."""
    import torch

    c1, _ = config1
    dm = pb.DeviceMatrix(sparse_from(c1), "float64")
    lab = torch.zeros(2000, dtype=torch.int32, device="cuda")
    lab[17] = 9
    torch.cuda.synchronize()
    with pytest.raises(ValueError):
        pcl.modularity_counts(dm, lab.data_ptr(), 4)
    lab[17] = 3
    torch.cuda.synchronize()
    intra, degsum = pcl.modularity_counts(dm, lab.data_ptr(), 4)
    assert degsum.sum() == dm.nnz
    dm.close()


@pytest.fixture(scope="module")
def cd():
    return load_golden("cli_downstream")


class TestCLIDownstream:
    """The reference CLI's `cluster` / `eval` commands on the device, against
    the reference CLI's own outputs (tests/golden/cli_downstream.npz)."""

    def _graph(self, cd, tmp_path):
        z, _ = cd
        g = tmp_path / "g.txt"
        g.write_text("\n".join(f"{u} {v}" for u, v in z["edges"]) + "\n")
        return str(g)

    def test_cluster(self, cd, tmp_path):
        import json

        from paper_1509_08360_b200 import cli

        z, meta = cd
        argv = list(meta["cluster"]["argv"])
        argv[argv.index("--input") + 1] = self._graph(cd, tmp_path)
        lab, summ = tmp_path / "labels.csv", tmp_path / "summary.json"
        assert cli.main(argv + ["--labels-out", str(lab), "--summary-out", str(summ)]) == 0
        got = json.load(open(summ))
        got.pop("input")
        assert got == meta["cluster"]["summary"]
        assert lab.read_bytes() == bytes(z["cluster_labels_csv"])

    def test_eval(self, cd, tmp_path):
        import csv
        import json

        from paper_1509_08360_b200 import cli
        from paper_1509_08360_b200 import io as pio

        z, meta = cd
        approx = tmp_path / "e.bin"
        pio.write_embedding(str(approx), z["eval_approx"])
        g = self._graph(cd, tmp_path)
        argv = ["eval", "--approx", str(approx), "--input", g] + meta["eval"]["argv_tail"][2:]
        pref = str(tmp_path / "ev")
        argv[argv.index("--output-prefix") + 1] = pref
        assert cli.main(argv) == 0
        rep, want = json.load(open(pref + "_report.json")), meta["eval"]["report"]
        assert (rep["pair_sample_size"], rep["zero_row_pairs"]) == (want["pair_sample_size"], want["zero_row_pairs"])
        for k, v in want["percentiles"].items():
            assert abs(rep["percentiles"][k] - v) <= 1e-10
        for part in ("percentiles", "calibration"):
            got = list(csv.reader(open(f"{pref}_{part}.csv")))
            ref = list(csv.reader(bytes(z[f"eval_{part}_csv"]).decode().splitlines()))
            assert got[0] == ref[0] and len(got) == len(ref)
            for gr, rr in zip(got[1:], ref[1:]):
                assert np.allclose([float(x) for x in gr], [float(x) for x in rr], rtol=0, atol=1e-10)
        # the same report from a precomputed exact embedding file
        ex = D.exact_embedding(pb.normalized_adjacency(z["edges"], 300).to_dense(), pb.indicator_above(0.5))
        exf = tmp_path / "exact.bin"
        pio.write_embedding(str(exf), ex.embedding)
        argv2 = ["eval", "--approx", str(approx), "--exact", str(exf), "--pairs", "5000", "--seed", "2",
                 "--output-prefix", pref + "2"]
        assert cli.main(argv2) == 0
        rep2 = json.load(open(pref + "2_report.json"))
        for k, v in want["percentiles"].items():
            assert abs(rep2["percentiles"][k] - v) <= 1e-10

    def test_eval_cap_exit_code(self, tmp_path):
        from paper_1509_08360_b200 import cli
        from paper_1509_08360_b200 import io as pio

        n = 3001
        g = tmp_path / "big.txt"
        g.write_text("\n".join(f"{i} {i + 1}" for i in range(n - 1)) + "\n")
        approx = tmp_path / "a.bin"
        pio.write_embedding(str(approx), np.ones((n, 4)))
        rc = cli.main(["eval", "--approx", str(approx), "--input", str(g), "--format", "edgelist", "--function",
                       "indicator:0.5", "--output-prefix", str(tmp_path / "x")])
        assert rc == 5


def test_fuzz_kmeans_modularity_cosines_vs_oracle():
    """Seeded random shapes: k-means labels / iteration counts / histories,
    modularity and pair cosines against the oracle (numpy restatement of the
    reference).  Covers d % 8 != 0, d < 8, d > 128, K not a multiple of the
    4-centroid quartet, ragged 64-row tiles and tight point clouds (empty clusters)."""
    rng = np.random.default_rng(2024)
    for case in range(24):
        n = int(rng.integers(2, 900))
        d = int(rng.choice([1, 3, 7, 8, 9, 16, 31, 40, 64, 80, 96, 127, 128, 129, 150]))
        K = int(rng.integers(1, min(n, 70) + 1))
        if case % 3 == 0:  # rows jittered around a few points (K > #points: empty clusters)
            # (exact duplicates are pinned by the reference's own fixture; at larger d
            # the reference's BLAS X @ C.T leaves ulp-level residues where the exact
            # answer is 0, so its seeding / reseed draws are BLAS-dependent there)
            pts = rng.standard_normal((max(1, K // 2), d))
            X = pts[rng.integers(0, len(pts), size=n)] + 1e-3 * rng.standard_normal((n, d))
        else:
            X = rng.standard_normal((n, d)) * rng.uniform(0.1, 10.0)
        seed = int(rng.integers(0, 2**31))
        a = pcl.kmeans(X, K, max_iters=40, seed=seed)
        labels, hist = O.kmeans(X, K, max_iters=40, seed=seed)
        assert np.array_equal(a.labels, labels), (case, n, d, K)
        _close_hist(a.inertia_history, hist, X)
        if n >= 3:
            m = max(1, int(rng.integers(1, 4 * n)))
            edges = rng.integers(0, n, size=(m, 2))
            if (edges[:, 0] != edges[:, 1]).any():
                q = pcl.modularity(edges, labels)
                want, mm = O.modularity(edges, labels)
                assert q.Q == want and q.m_edges == mm
            pairs = D.sample_pairs(n, min(500, n * (n - 1) // 2), case)
            cos, _ = D.pair_correlations(X, pairs)
            assert np.max(np.abs(cos - O.pair_cosines(X, pairs))) <= COS_ABS


def test_large_k_global_counts():
    """K above the 16384-cluster shared-histogram limit: counts and the
    counting sort switch to global atomics; ~1 point per cluster also drives
    thousands of empty-cluster reseeds per iteration."""
    rng = np.random.default_rng(77)
    X = rng.standard_normal((17_000, 3))
    a = pcl.kmeans(X, 16_500, max_iters=2, seed=5)
    labels, hist = O.kmeans(X, 16_500, max_iters=2, seed=5)
    assert np.array_equal(a.labels, labels)
    _close_hist(a.inertia_history, hist, X)


def test_nan_and_overflow_rows_follow_the_reference():
    """Non-finite rows: the ++ seeding raises numpy's `Probabilities contain NaN`
    (rng.choice) like the reference; with K=1 (no weighted pick) NaN flows
    through Lloyd as in numpy (argmin treats NaN as the minimum)."""
    rng = np.random.default_rng(0)
    X = rng.standard_normal((50, 4))
    X[7] = np.nan
    with pytest.raises(ValueError, match="Probabilities contain NaN"):
        pcl.kmeans(X, 3, seed=1)
    Y = rng.standard_normal((50, 4))
    Y[7, 0] = 1e200  # |x|^2 overflows to inf
    with pytest.raises(ValueError, match="Probabilities contain NaN"):
        pcl.kmeans(Y, 3, seed=1)
    a = pcl.kmeans(X, 1, seed=1)
    labels, hist = O.kmeans(X, 1, seed=1)
    assert np.array_equal(a.labels, labels)
    assert len(a.inertia_history) == len(hist) and all(np.isnan(a.inertia_history)) == all(np.isnan(hist))


def test_distance_bound_audit_vs_reference():
    """oracle.distance_bound_audit on the device (cuSOLVER spectrum, device seam
    embeddings, fp64 device distances) vs the reference's fractions
    (tests/golden/audit.npz); pairs within ulps of a bound may flip (<= 3)."""
    z, meta = load_golden("audit")
    S = pb.scale_values(pb.normalized_adjacency(z["edges"], 300), 0.98)
    n_pairs = 300 * 299 // 2
    for name, m in meta.items():
        cfg = pb.EmbedConfig(L=m["L"], d=m["d"], seed=m["seed"], epsilon=m["epsilon"])
        got = D.distance_bound_audit(S, pb.parse_function(m["function"]), cfg, m["trials"])
        assert abs(got - m["fraction"]) * m["trials"] * n_pairs <= 3, (name, got, m["fraction"])
