"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

This script is the only place that imports the reference package (`csemb`,
read-only at /root/reference/pkg/src). It runs in the build container, where
the reference is importable, and writes small .npz fixtures that travel with
the repo; nothing on the GPU box reads /root/reference.

    python tests/golden/make_golden.py          # rewrites tests/golden/*.npz

Every fixture records the reference call that produced it (see `CASES` below
and the `meta` string inside each file).
"""

from __future__ import annotations

import hashlib
import json
import logging
import os
import re
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.dirname(os.path.abspath(__file__))

sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.dont_write_bytecode = True

import csemb as cs  # noqa: E402  (reference, read-only)
from csemb import engine as ref_engine  # noqa: E402
from helpers import random_symmetric, sbm  # noqa: E402  (reference test helpers)


class _StepLog(logging.Handler):
    """Collect the reference's per-step debug records (engine.py:218-220)."""

    pat = re.compile(r"stage=(\d+) cols=(\d+)\+(\d+) r=(\d+) max_abs=(\S+)")

    def __init__(self):
        super().__init__(logging.DEBUG)
        self.rows = []

    def emit(self, record):
        m = self.pat.match(record.getMessage())
        if m:
            st, c0, w, r, peak = m.groups()
            self.rows.append((int(st), int(c0), int(w), int(r), float(peak)))


def _capture():
    h = _StepLog()
    lg = logging.getLogger("csemb.engine")
    lg.setLevel(logging.DEBUG)
    lg.addHandler(h)
    return h, lg


def _csr(S):
    return dict(
        n_rows=np.int64(S.n_rows),
        n_cols=np.int64(S.n_cols),
        row_offsets=np.asarray(S.row_offsets, dtype=np.int64),
        col_indices=np.asarray(S.col_indices, dtype=np.int32),
        values=np.asarray(S.values, dtype=np.float64),
    )


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _save(name, meta, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, meta=np.array(json.dumps(meta, sort_keys=True)), **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


class CutAbove:
    """f(x) = x * 1{x >= c} (config 4's PCA-like weight); a plain callable with
    breakpoints, used identically by both sides."""

    def __init__(self, c):
        self.c = float(c)

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        return np.where(x >= self.c, x, 0.0)

    def breakpoints(self):
        return (self.c,)


def gen_omega():
    cases = [(3, 4, 42), (50, 9, 3), (40, 7, 11), (40, 80, 0), (2000, 40, 0), (1000, 96, 123456789)]
    arrays = {}
    for n, d, seed in cases:
        om = cs.sample_projection(n, d, seed)
        arrays[f"signs_{n}_{d}_{seed}"] = np.packbits(om > 0, axis=None)
    folds = np.array(
        [cs.fold_seed(s, t) for s, t in [(0, 0x6E6F726D), (13, 0), (2024, 5), (2**63 + 7, 3)]],
        dtype=np.uint64,
    )
    _save(
        "omega",
        {"call": "csemb.sample_projection(n,d,seed) > 0, packbits; fold_seed", "cases": cases,
         "fold_cases": [(0, 0x6E6F726D), (13, 0), (2024, 5), (2**63 + 7, 3)]},
        folds=folds,
        **arrays,
    )


def gen_config1():
    """BASELINE config 1: SBM n=2000, 4 blocks, p_in .05, p_out .005, graph seed 0,
    d=40 (seed 0), f = 1{x >= 0.9}, L=60, fp64."""
    edges, labels = sbm(2000, 4, 0.05, 0.005, np.random.default_rng(0))
    S = cs.normalized_adjacency(edges, 2000)
    omega = cs.sample_projection(2000, 40, 0)
    f = cs.indicator_above(0.9)
    h, lg = _capture()
    emb = cs.fast_embed_eig(S, f, 60, omega)
    lg.removeHandler(h)
    exp = cs.legendre_coefficients(f, 60)
    steps = np.array([(r, c0, peak) for (_, c0, _, r, peak) in h.rows], dtype=np.float64)
    pairs = cs.sample_pairs(2000, 10_000, 0)
    norm_est = cs.estimate_spectral_norm(S, cs.EmbedConfig(L=60, d=40, seed=0))
    _save(
        "config1",
        {
            "call": "fast_embed_eig(normalized_adjacency(sbm(2000,4,.05,.005,rng0)), indicator_above(0.9), 60, sample_projection(2000,40,0))",
            "provenance": emb.provenance,
            "E_sha256": _sha(emb.values),
            "E_fro": float(np.linalg.norm(emb.values)),
            "norm_estimate": norm_est,
        },
        edges=edges.astype(np.int32),
        labels=labels.astype(np.int32),
        coeffs=exp.coeffs,
        E=emb.values,
        step_max_abs=steps,
        pairs=pairs.astype(np.int32),
        **_csr(S),
    )


def gen_small_cases():
    """Small engine cases: cascade, general (dilation), worker/column-subset,
    polynomial exactness, divergence.  Inputs are stored as CSR so the device
    side needs no generator."""
    out = {}
    meta = {}

    # cascade b=2 vs the reference (tests/test_engine.py:201-215 setup)
    dense = random_symmetric(80, np.random.default_rng(13), spectral_norm=0.98)
    S = cs.SparseMatrix.from_dense(dense)
    cfg = cs.EmbedConfig(L=180, d=8, b=2, seed=13)
    om = cs.sample_projection(80, 8, 13)
    counter = cs.SpmvCounter()
    emb = cs.fast_embed_cascaded(S, cs.indicator_above(0.98), cfg, om, counter=counter)
    for k, v in _csr(S).items():
        out[f"cascade_{k}"] = v
    out["cascade_E"] = emb.values
    meta["cascade"] = {"call": "fast_embed_cascaded(S80, indicator_above(.98), EmbedConfig(L=180,d=8,b=2,seed=13), sample_projection(80,8,13))",
                       "provenance": emb.provenance}

    # rectangular general path, b=2 (tests/test_engine.py:243-265 setup)
    rng = np.random.default_rng(18)
    A = rng.standard_normal((7, 5))
    A /= np.linalg.norm(A, 2) * 1.02
    As = cs.SparseMatrix.from_dense(A)
    cfg = cs.EmbedConfig(L=80, d=9, b=2, seed=18)
    rows, cols = cs.fast_embed_general(As, cs.indicator_above(0.4), cfg)
    for k, v in _csr(As).items():
        out[f"general_{k}"] = v
    out["general_rows"] = rows.values
    out["general_cols"] = cols.values
    meta["general"] = {"call": "fast_embed_general(A7x5, indicator_above(.4), EmbedConfig(L=80,d=9,b=2,seed=18))",
                       "provenance": rows.provenance}

    # sparse rectangular, b=1, config-4-like weight (odd extension of x*1{x>=.3})
    rng = np.random.default_rng(44)
    m, n = 300, 120
    Ad = rng.random((m, n)) * (rng.random((m, n)) < 0.05)
    Ad /= np.linalg.norm(Ad, 2) * 1.01
    As = cs.SparseMatrix.from_dense(Ad)
    cfg = cs.EmbedConfig(L=120, d=24, b=1, seed=4)
    rows, cols = cs.fast_embed_general(As, CutAbove(0.3), cfg)
    for k, v in _csr(As).items():
        out[f"general2_{k}"] = v
    out["general2_rows"] = rows.values
    out["general2_cols"] = cols.values
    out["general2_dilated_row_offsets"] = np.asarray(cs.dilate(As).row_offsets)
    out["general2_dilated_col_indices"] = np.asarray(cs.dilate(As).col_indices, dtype=np.int32)
    out["general2_dilated_values"] = np.asarray(cs.dilate(As).values)
    meta["general2"] = {"call": "fast_embed_general(A300x120 sparse, CutAbove(0.3), EmbedConfig(L=120,d=24,seed=4))",
                        "provenance": rows.provenance}

    # column-chunk crossing width, odd d (d=70 crosses two 32-col chunks)
    dense = random_symmetric(50, np.random.default_rng(10))
    S = cs.SparseMatrix.from_dense(dense)
    om = cs.sample_projection(50, 70, 10)
    h, lg = _capture()
    emb = cs.fast_embed_eig(S, cs.indicator_above(0.0), 12, om, n_workers=4)
    lg.removeHandler(h)
    for k, v in _csr(S).items():
        out[f"wide_{k}"] = v
    out["wide_E"] = emb.values
    out["wide_steps"] = np.array(sorted((r, c0, peak) for (_, c0, _, r, peak) in h.rows), dtype=np.float64)
    meta["wide"] = {"call": "fast_embed_eig(S50, indicator_above(0), 12, sample_projection(50,70,10), n_workers=4)"}

    # polynomial exactness input (tests/test_engine.py:119-130, seed 0)
    rng = np.random.default_rng(100)
    dense = random_symmetric(150, rng, density=0.1, spectral_norm=0.97)
    coeffs = rng.standard_normal(6)
    S = cs.SparseMatrix.from_dense(dense)
    om = cs.sample_projection(150, 10, 0)
    emb = cs.fast_embed_eig(S, lambda x: np.polynomial.polynomial.polyval(x, coeffs), 5, om)
    for k, v in _csr(S).items():
        out[f"poly_{k}"] = v
    out["poly_monomial"] = coeffs
    out["poly_E"] = emb.values
    out["poly_theta"] = cs.legendre_coefficients(lambda x: np.polynomial.polynomial.polyval(x, coeffs), 5).coeffs
    meta["poly"] = {"call": "fast_embed_eig(S150, polyval(coeffs), 5, sample_projection(150,10,0))"}

    # divergence (tests/test_engine.py:173-177)
    S = cs.SparseMatrix.from_dense(10.0 * np.eye(4))
    om = cs.sample_projection(4, 2, 0)
    try:
        cs.fast_embed_eig(S, cs.identity(), 250, om)
        raise SystemExit("reference did not diverge")
    except cs.DivergenceError as exc:
        r = int(re.search(r"r=(\d+)", str(exc)).group(1))
        meta["divergence"] = {"first_bad_r": r, "message": str(exc)}
    _save("small_cases", meta, **out)


def gen_coefficients():
    specs = {
        "ind090_60": (cs.indicator_above(0.9), 60),
        "ind095_180": (cs.indicator_above(0.95), 180),
        "commute001_180": (cs.commute_time(0.01), 180),
        "cut030_odd_120": (cs.odd_extension(CutAbove(0.3)), 120),
        "ind098_root2_90": (cs.root_function(cs.indicator_above(0.98), 2), 90),
        "ind040_odd_root2_40": (cs.odd_extension(cs.root_function(cs.indicator_above(0.4), 2)), 40),
        "identity_1": (cs.identity(), 1),
        "identity_7": (cs.identity(), 7),
        "const25_0": (cs.constant(2.5), 0),
        "table_33": (cs.tabulated([-1.0, -0.2, 0.5, 1.0], [0.0, 1.0, -0.5, 2.0]), 33),
        "ind09_odd_60": (cs.odd_extension(cs.indicator_above(0.9)), 60),
        "commute_root3_30": (cs.root_function(cs.commute_time(0.05), 3), 30),
    }
    arrays, meta = {}, {}
    for name, (f, order) in specs.items():
        e = cs.legendre_coefficients(f, order)
        arrays[name] = e.coeffs
        meta[name] = {"describe": getattr(f, "describe", lambda: "callable")(), "sha256": e.digest()}
    _save("coefficients", meta, **arrays)


def gen_norm():
    arrays, meta = {}, {}
    cases = {}
    cases["identity10"] = (cs.SparseMatrix.identity(10), cs.EmbedConfig(L=1, d=1, seed=0))
    dense = np.zeros((50, 50))
    dense[0, 0], dense[1, 1] = 0.3, -0.9
    cases["paddiag"] = (cs.SparseMatrix.from_dense(dense), cs.EmbedConfig(L=1, d=1, seed=1))
    for seed in range(3):
        dense = random_symmetric(60, np.random.default_rng(seed), spectral_norm=None)
        cases[f"rand60_{seed}"] = (cs.SparseMatrix.from_dense(dense), cs.EmbedConfig(L=1, d=1, seed=seed))
    rng = np.random.default_rng(7)
    A = rng.random((90, 40)) * (rng.random((90, 40)) < 0.1)
    cases["dilated90x40_30it"] = (cs.dilate(cs.SparseMatrix.from_dense(A)), cs.EmbedConfig(L=1, d=1, seed=3, norm_iters=30))
    for name, (S, cfg) in cases.items():
        est = cs.estimate_spectral_norm(S, cfg)
        for k, v in _csr(S).items():
            arrays[f"{name}_{k}"] = v
        meta[name] = {"estimate": est, "seed": cfg.seed, "norm_iters": cfg.norm_iters,
                      "norm_vectors_factor": cfg.norm_vectors_factor, "norm_safety": cfg.norm_safety,
                      "exact_norm": float(np.linalg.norm(S.to_dense(), 2))}
    _save("norm", meta, **arrays)


def gen_builders():
    arrays, meta = {}, {}
    rng = np.random.default_rng(5)
    for i, (n, m) in enumerate([(2, 1), (3, 4), (30, 120), (500, 3000)]):
        edges = rng.integers(0, n, size=(m, 2))
        S = cs.normalized_adjacency(edges, n)
        arrays[f"adj{i}_edges"] = edges.astype(np.int64)
        for k, v in _csr(S).items():
            arrays[f"adj{i}_{k}"] = v
        meta[f"adj{i}"] = {"n": n}
    A = cs.SparseMatrix.from_dense(np.random.default_rng(6).random((6, 9)) * (np.random.default_rng(7).random((6, 9)) < 0.4))
    D = cs.dilate(A)
    for k, v in _csr(A).items():
        arrays[f"dil_A_{k}"] = v
    for k, v in _csr(D).items():
        arrays[f"dil_S_{k}"] = v
    _save("builders", meta, **arrays)


def gen_cli():
    """The reference CLI (cli.py main) on three small inputs: an edge list
    (normalized adjacency, cascade b=2), a raw symmetric Matrix Market matrix
    (norm-estimate rescaling) and a rectangular one (dilation)."""
    import tempfile

    import scipy.io
    import scipy.sparse as sp
    from csemb import io as cio
    from csemb.cli import main

    arrays, meta = {}, {}
    edges, _ = sbm(120, 4, 0.3, 0.02, np.random.default_rng(88))
    rng = np.random.default_rng(9)
    raw = random_symmetric(60, rng, density=0.15, spectral_norm=None) * 3.0
    rect = rng.random((40, 25)) * (rng.random((40, 25)) < 0.3)
    arrays["edges"] = edges.astype(np.int64)
    arrays["raw"] = raw
    arrays["rect"] = rect
    drop = ("wall_time_s", "input", "output")
    with tempfile.TemporaryDirectory() as tmp:
        g = os.path.join(tmp, "g.txt")
        with open(g, "w") as fh:
            fh.write("\n".join(f"{u} {v}" for u, v in edges) + "\n")
        scipy.io.mmwrite(os.path.join(tmp, "raw.mtx"), sp.coo_array(raw))
        scipy.io.mmwrite(os.path.join(tmp, "rect.mtx"), sp.coo_array(rect))
        runs = {
            "edgelist": ["embed", "--input", g, "--format", "edgelist", "--matrix", "normalized-adjacency",
                         "--function", "indicator:0.3", "--L", "48", "--b", "2", "--d", "40", "--seed", "123"],
            "raw": ["embed", "--input", os.path.join(tmp, "raw.mtx"), "--format", "matrix-market",
                    "--matrix", "raw", "--function", "indicator:0.2", "--L", "20", "--d", "16", "--seed", "5"],
            "dilation": ["embed", "--input", os.path.join(tmp, "rect.mtx"), "--format", "matrix-market",
                         "--matrix", "dilation", "--function", "indicator:0.3", "--L", "30", "--d", "12",
                         "--seed", "6"],
        }
        for name, argv in runs.items():
            out = os.path.join(tmp, name + ".bin")
            cols = os.path.join(tmp, name + ".cols.bin")
            extra = ["--output-cols", cols] if name == "dilation" else []
            assert main(argv + ["--output", out] + extra) == 0
            with open(out, "rb") as fh:
                blob = fh.read()
            arrays[f"{name}_E"] = cio.read_embedding(out)
            if extra:
                arrays[f"{name}_cols"] = cio.read_embedding(cols)
            md = json.load(open(out + ".meta.json"))
            meta[name] = {"argv": argv, "sha256": hashlib.sha256(blob).hexdigest(),
                          "metadata": {k: v for k, v in md.items() if k not in drop}}
        ns = os.path.join(tmp, "norm.json")
        assert main(["norm", "--input", os.path.join(tmp, "raw.mtx"), "--format", "matrix-market", "--matrix", "raw",
                     "--seed", "3", "--output", ns]) == 0
        meta["norm"] = json.load(open(ns))
    _save("cli", meta, **arrays)


def _dup_points():
    """30 rows on 5 distinct points: with K=8 the ++ seeding runs out of
    positive distance (total <= 0 branch) and Lloyd meets empty clusters."""
    rng = np.random.default_rng(17)
    base = rng.standard_normal((5, 6))
    return base[rng.integers(0, 5, size=30)]


def _blobs(n, d, k, seed):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, d)) * 4.0
    return centers[rng.integers(0, k, size=n)] + rng.standard_normal((n, d))


def gen_downstream():
    """Downstream consumers: cluster.kmeans, cluster.modularity,
    cluster.cluster_experiment, oracle._pair_correlations and
    oracle.distortion_percentiles on the config-1 embedding, plus k-means on
    Gaussian blobs (K=70: two centroid tiles) and on duplicated points."""
    from csemb import cluster as ccl
    from csemb import oracle as cor

    edges, labels = sbm(2000, 4, 0.05, 0.005, np.random.default_rng(0))
    S = cs.normalized_adjacency(edges, 2000)
    f = cs.indicator_above(0.9)
    emb = cs.fast_embed_eig(S, f, 60, cs.sample_projection(2000, 40, 0))
    E = emb.values
    arrays, meta = {}, {"kmeans": {}, "modularity": {}}
    inputs = {"config1": E, "blobs": _blobs(3000, 20, 70, 5), "dup": _dup_points()}
    arrays["blobs_X"] = inputs["blobs"]
    arrays["dup_X"] = inputs["dup"]
    cases = [("config1", 4, 0x6B6D6531), ("config1", 4, 0x6B6D6532), ("config1", 9, 7),
             ("blobs", 70, 11), ("blobs", 3, 2), ("dup", 8, 4), ("dup", 1, 0)]
    for name, K, seed in cases:
        km = ccl.kmeans(inputs[name], K, seed=seed)
        key = f"{name}_K{K}_s{seed}"
        arrays[f"km_{key}_labels"] = km.labels.astype(np.int16)
        arrays[f"km_{key}_history"] = np.array(km.inertia_history)
        meta["kmeans"][key] = {"input": name, "K": K, "seed": seed, "n_iters": km.n_iters,
                               "inertia": km.inertia}
        if name == "config1":
            q = ccl.modularity(edges, km)
            meta["modularity"][key] = {"Q": q.Q, "m_edges": q.m_edges}
    q = ccl.modularity(edges, labels)
    meta["modularity"]["truth"] = {"Q": q.Q, "m_edges": q.m_edges}
    ex = ccl.cluster_experiment(edges, 2000, f, cs.EmbedConfig(L=60, d=40, seed=0), K=4, runs=5)
    meta["experiment"] = {"call": "cluster_experiment(edges, 2000, indicator_above(0.9), EmbedConfig(L=60,d=40,seed=0), K=4, runs=5)",
                          "median_modularity": ex.median_modularity, "run_scores": list(ex.run_scores)}
    arrays["experiment_median_labels"] = ex.median_labels.astype(np.int16)
    pairs = cs.sample_pairs(2000, 10_000, 0)
    cos, zero = cor._pair_correlations(E, pairs)
    arrays["pair_cos"] = cos
    exact = cor.exact_embedding(S, f)
    arrays["exact_embedding"] = exact.embedding
    for mode in ("deviation", "calibration"):
        rep = cor.distortion_percentiles(exact, emb, n_pairs=20_000, seed=3, mode=mode)
        meta[f"distortion_{mode}"] = cor.report_to_dict(rep)
    meta["distortion_call"] = "distortion_percentiles(exact_embedding(S, f), emb, n_pairs=20000, seed=3, mode)"
    _save("downstream", meta, **arrays)


def gen_cli_downstream():
    """The reference CLI's `cluster` and `eval` commands (cli.py:226-281) on a
    small SBM edge list: cluster summary JSON + labels CSV; eval's percentile /
    calibration CSVs and report JSON for an embedding from its own `embed`."""
    import tempfile

    from csemb.cli import main

    edges, _ = sbm(300, 3, 0.2, 0.01, np.random.default_rng(41))
    arrays, meta = {"edges": edges.astype(np.int64)}, {}
    with tempfile.TemporaryDirectory() as tmp:
        g = os.path.join(tmp, "g.txt")
        with open(g, "w") as fh:
            fh.write("\n".join(f"{u} {v}" for u, v in edges) + "\n")
        cl = ["cluster", "--input", g, "--function", "indicator:0.5", "--L", "40", "--d", "24", "--seed", "5",
              "--k", "3", "--runs", "5"]
        lab, summ = os.path.join(tmp, "labels.csv"), os.path.join(tmp, "summary.json")
        assert main(cl + ["--labels-out", lab, "--summary-out", summ]) == 0
        meta["cluster"] = {"argv": cl, "summary": json.load(open(summ))}
        meta["cluster"]["summary"].pop("input")
        arrays["cluster_labels_csv"] = np.frombuffer(open(lab, "rb").read(), dtype=np.uint8)
        emb = os.path.join(tmp, "e.bin")
        em = ["embed", "--input", g, "--format", "edgelist", "--function", "indicator:0.5", "--L", "40",
              "--d", "24", "--seed", "5", "--output", emb]
        assert main(em) == 0
        arrays["eval_approx"] = cio_read(emb)
        ev = ["eval", "--approx", emb, "--input", g, "--format", "edgelist", "--function", "indicator:0.5",
              "--pairs", "5000", "--seed", "2", "--output-prefix", os.path.join(tmp, "ev")]
        assert main(ev) == 0
        meta["eval"] = {"argv_tail": ev[3:], "report": json.load(open(os.path.join(tmp, "ev_report.json")))}
        for part in ("percentiles", "calibration"):
            arrays[f"eval_{part}_csv"] = np.frombuffer(open(os.path.join(tmp, f"ev_{part}.csv"), "rb").read(),
                                                       dtype=np.uint8)
    _save("cli_downstream", meta, **arrays)


def cio_read(path):
    from csemb import io as cio

    return cio.read_embedding(path)


def gen_audit():
    """oracle.distance_bound_audit (oracle.py:196-216): the violation fraction
    for two settings on a small SBM (n=300, normalized adjacency scaled by 0.98)."""
    from csemb import oracle as cor

    edges, _ = sbm(300, 3, 0.2, 0.01, np.random.default_rng(41))
    S = cs.scale_values(cs.normalized_adjacency(edges, 300), 0.98)  # spectrum strictly inside [-1, 1]
    # (L, d, epsilon, trials, function): the identity is represented exactly
    # (delta ~ 1e-16), so at small d the JL band is violated for a real share of pairs
    cases = {"indicator": (40, 24, 0.5, 3, "indicator:0.5"), "identity_d8": (4, 8, 0.2, 3, "identity"),
             "identity_d24": (6, 24, 0.3, 2, "identity")}
    meta = {}
    for name, (L, d, eps, trials, spec) in cases.items():
        cfg = cs.EmbedConfig(L=L, d=d, seed=9, epsilon=eps)
        f = cs.parse_function(spec)
        meta[name] = {"L": L, "d": d, "epsilon": eps, "trials": trials, "function": spec, "seed": 9,
                      "fraction": cor.distance_bound_audit(S, f, cfg, trials)}
    _save("audit", meta, edges=edges.astype(np.int64))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_omega()
    gen_config1()
    gen_small_cases()
    gen_coefficients()
    gen_norm()
    gen_builders()
    gen_cli()
    gen_downstream()
    gen_cli_downstream()
    gen_audit()
