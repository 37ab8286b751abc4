"""Downstream consumers, CPU side: the oracle's k-means and
modularity restatements pinned bit-for-bit to the reference's fixtures
(tests/golden/downstream.npz from make_golden.py), and the product's host
logic (pair sampling, distortion binning / percentiles / writers, the k-means
control flow driven by a numpy stand-in for the device steps)."""

import csv
import json

import numpy as np
import pytest

import oracle as O
from oracle.oracle import _sqdist
from conftest import load_golden
from paper_1509_08360_b200 import cluster as pcl
from paper_1509_08360_b200 import distortion as D


@pytest.fixture(scope="module")
def ds():
    return load_golden("downstream")


@pytest.fixture(scope="module")
def rows(ds, config1):
    z, _ = ds
    c1, _ = config1
    return {"config1": c1["E"], "blobs": z["blobs_X"], "dup": z["dup_X"]}


def test_oracle_kmeans_matches_reference(ds, rows):
    z, meta = ds
    for key, m in meta["kmeans"].items():
        labels, hist = O.kmeans(rows[m["input"]], m["K"], seed=m["seed"])
        assert np.array_equal(labels, z[f"km_{key}_labels"]), key
        assert np.array_equal(np.array(hist), z[f"km_{key}_history"]), key
        assert len(hist) == m["n_iters"]


def test_oracle_modularity_matches_reference(ds, config1):
    z, meta = ds
    c1, _ = config1
    q, m = O.modularity(c1["edges"], c1["labels"])
    assert (q, m) == (meta["modularity"]["truth"]["Q"], meta["modularity"]["truth"]["m_edges"])
    for key, want in meta["modularity"].items():
        if key == "truth":
            continue
        q, m = O.modularity(c1["edges"], z[f"km_{key}_labels"])
        assert q == want["Q"] and m == want["m_edges"]


def test_sample_pairs_matches_reference(config1):
    c1, _ = config1
    assert np.array_equal(D.sample_pairs(2000, 10_000, 0), c1["pairs"])
    for n, k, s in [(50, 1225, 3), (50, 1000, 2), (10, None, 1), (100_000, 5000, 9), (3, 2, 0), (2, 5, 0)]:
        assert np.array_equal(D.sample_pairs(n, k, s), O.sample_pairs(n, k if k is not None else 100_000, s))


def test_distortion_host_logic_matches_reference(ds, config1, monkeypatch, tmp_path):
    """With the reference's own correlations substituted for the device pass,
    the report is identical to the reference's (binning, percentiles, JSON)."""
    z, meta = ds
    c1, _ = config1

    def corr(rows, pairs, *, device=0):
        rows = D._rows(rows)
        nr = np.linalg.norm(rows, axis=1)
        den = nr[pairs[:, 0]] * nr[pairs[:, 1]]
        out = np.zeros(len(pairs))
        dots = np.einsum("ij,ij->i", rows[pairs[:, 0]], rows[pairs[:, 1]])
        np.divide(dots, den, out=out, where=den != 0)
        return out, den == 0

    monkeypatch.setattr(D, "pair_correlations", corr)
    for mode in ("deviation", "calibration"):
        rep = D.distortion_percentiles(z["exact_embedding"], c1["E"], n_pairs=20_000, seed=3, mode=mode)
        assert D.report_to_dict(rep) == meta[f"distortion_{mode}"]
        D.write_report_json(rep, tmp_path / f"{mode}.json")
        assert json.load(open(tmp_path / f"{mode}.json")) == meta[f"distortion_{mode}"]
        if mode == "deviation":
            D.write_percentiles_csv(rep, tmp_path / "p.csv")
            got = list(csv.reader(open(tmp_path / "p.csv")))
            assert got[0] == ["percentile", "value"] and len(got) == 8
            with pytest.raises(ValueError):
                D.write_calibration_csv(rep, tmp_path / "c.csv")
        else:
            D.write_calibration_csv(rep, tmp_path / "c.csv")
            got = list(csv.reader(open(tmp_path / "c.csv")))
            assert got[0][0] == "bin_center" and len(got) == 1 + len(rep.bins)
    with pytest.raises(ValueError):
        D.distortion_percentiles(c1["E"], c1["E"][:10], mode="deviation")
    with pytest.raises(ValueError):
        D.distortion_percentiles(c1["E"], c1["E"], mode="bogus")


class _NumpyKMeans:
    """Stand-in for DeviceKMeans with the reference's numpy arithmetic: drives
    the product's host loop (cluster._run_kmeans) without a GPU."""

    def __init__(self, X, K):
        self.X, self.K, self.n = np.asarray(X, np.float64), K, len(X)
        self.C = np.zeros((K, self.X.shape[1]))
        self.lab = np.full(self.n, -1)

    def seed(self, k, row):
        self.C[k] = self.X[row]
        d2 = _sqdist(self.X, self.C[k:k + 1])[:, 0]
        self.closest = d2 if k == 0 else np.minimum(self.closest, d2)
        return float(self.closest.sum())

    def pick(self, u):
        p = self.closest / self.closest.sum()
        cdf = p.cumsum()
        cdf /= cdf[-1]
        return int(cdf.searchsorted(u, side="right"))

    def assign(self):
        d2 = _sqdist(self.X, self.C)
        self.new = np.argmin(d2, axis=1)
        self.mind = d2[np.arange(self.n), self.new]
        return float(self.mind.sum()), int(np.sum(self.new != self.lab)), np.bincount(self.new, minlength=self.K)

    def reseed(self, c):
        far = int(np.argmax(self.mind))
        self.C[c], self.new[far], self.mind[far] = self.X[far], c, -1.0
        return far

    def commit(self, update):
        self.lab = self.new.copy()
        if update:
            acc = np.zeros_like(self.C)
            np.add.at(acc, self.lab, self.X)
            self.C = acc / np.bincount(self.lab, minlength=self.K)[:, None]

    def labels(self):
        return self.lab.astype(np.int64)


def test_host_loop_replays_reference_control_flow(ds, rows):
    """cluster._run_kmeans (the product's loop) with numpy device steps gives
    the reference's labels and history exactly: draw order, branches and
    empty-cluster handling are the reference's."""
    z, meta = ds
    for key, m in meta["kmeans"].items():
        a = pcl._run_kmeans(_NumpyKMeans(rows[m["input"]], m["K"]), m["K"], 100, m["seed"])
        assert np.array_equal(a.labels, z[f"km_{key}_labels"]), key
        assert np.array_equal(np.array(a.inertia_history), z[f"km_{key}_history"]), key
        assert a.n_iters == m["n_iters"] and a.inertia == m["inertia"]


def test_modularity_score_expression():
    s = pcl._score(np.array([3, 1]), np.array([8.0, 6.0]), 7)
    assert s.Q == float(np.sum(np.array([3, 1]) / 7 - (np.array([8.0, 6.0]) / 14.0) ** 2))
    with pytest.raises(ValueError):
        pcl.ModularityScore(Q=1.5, m_edges=1)
