"""Generate golden vectors by running the REAL reference package.

Run in the build container only (the reference tree is not on the GPU box):

    python tests/golden/make_golden.py            # all small fixtures
    python tests/golden/make_golden.py --c1       # + the full config-1 run (~2 min)

The reference is imported from /root/reference/pkg/src under the alias
``speclust_ref`` so it cannot collide with anything in this repo.  Outputs are
written next to this script as compressed .npz files.  Large arrays of the
config-1 run are stored as SHA-256 digests (bit-exact structure checks) plus
the small per-node vectors.
"""

from __future__ import annotations

import argparse
import hashlib
import importlib.util
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src/speclust/__init__.py")


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "speclust_ref", REF_SRC, submodule_search_locations=[str(REF_SRC.parent)]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["speclust_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def blobs(n, d, k, cs, seed=0):
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, cs, (k, d))
    y = rng.integers(0, k, n)
    return np.ascontiguousarray(centers[y] + rng.standard_normal((n, d))), y


def chosen_rows(v, init_c):
    """Recover k-means++ row indices from the coordinates the reference returns."""
    lut = {v[i].tobytes(): i for i in range(v.shape[0])}
    return np.array([lut[r.tobytes()] for r in init_c], dtype=np.int64)


def graph_case(sp, x, knn, sigma):
    m = sp.SimilarityMeasure.exp_decay(sigma)
    e = sp.build_edges_knn(x, knn, m)
    w = sp.coo_to_csr(sp.build_similarity(x, e, m))
    d = sp.degrees(w)
    sym = sp.sym_scale(w, d).vals if np.all(d > 0.0) else np.zeros(0)
    return dict(edges=e, row_ptr=w.row_ptr, col=w.col_idx, vals=w.vals, degrees=d,
                sym_vals=sym)


def pipeline_case(sp, x, knn, sigma, k, timing=False):
    cfg = sp.PipelineConfig(
        input=sp.PointsInput(measure=sp.SimilarityMeasure.exp_decay(sigma), pattern="knn",
                             points=x, knn=knn),
        k_clusters=k,
        eigen=sp.LanczosConfig(k=k, seed=0),
        kmeans=sp.KmeansConfig(k=k, seed=0),
        normalize_rows=True,
    )
    t0 = time.perf_counter()
    rep = sp.run(cfg)
    wall = time.perf_counter() - t0
    # re-derive the intermediate arrays with the reference's own stage calls
    g = graph_case(sp, x, knn, sigma)
    w = sp.CsrMatrix(len(x), len(x), g["row_ptr"], g["col"], g["vals"])
    a = sp.sym_scale(w, g["degrees"])
    basis = sp.eigensolve(a, sp.LanczosConfig(k=k, seed=0))
    emb = sp.recover_row_eigvecs(basis.vectors, g["degrees"])
    norms = np.linalg.norm(emb, axis=1, keepdims=True)
    norms[norms == 0.0] = 1.0
    rows = emb / norms
    init_c = sp.kmeanspp_init(rows, k, 0)
    out = dict(g)
    out.update(values=basis.values, vectors=basis.vectors, residuals=basis.residuals,
               embedding=rows, chosen=chosen_rows(rows, init_c),
               labels=rep.labeling.labels, centroids=rep.labeling.centroids,
               sse=rep.labeling.sse, iters=rep.labeling.iters_run,
               sse_history=rep.labeling.sse_history, ncut=rep.ncut_value,
               report_values=rep.eigenvalues, wall=wall)
    for key, val in rep.timings.items():
        out["t_" + key] = val
    assert np.array_equal(rep.eigenvalues, basis.values)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", action="store_true", help="also run full config 1 (N=20k)")
    args = ap.parse_args()
    sp = load_reference()
    rng = np.random.default_rng(20260417)

    # ---- graph fixtures -------------------------------------------------
    x, _ = blobs(600, 8, 6, 2.0, seed=1)
    np.savez_compressed(HERE / "graph_blobs600.npz", x=x, knn=6, sigma=np.sqrt(8.0),
                        **graph_case(sp, x, 6, np.sqrt(8.0)))
    # underflow ties: 4 points 100 apart, sigma 0.5, knn 1
    x = np.array([[0.0], [100.0], [200.0], [300.0]])
    np.savez_compressed(HERE / "graph_underflow.npz", x=x, knn=1, sigma=0.5,
                        **graph_case(sp, x, 1, 0.5))
    # duplicated points + integer lattice (exact ties in d2)
    base = rng.integers(0, 4, (150, 3)).astype(np.float64)
    x = np.concatenate((base, base[:40]))
    np.savez_compressed(HERE / "graph_ties.npz", x=x, knn=5, sigma=1.3,
                        **graph_case(sp, x, 5, 1.3))
    # C2-shape at small N (d=64, kNN=32, cs=0.7)
    x, _ = blobs(3000, 64, 100, 0.7, seed=2)
    np.savez_compressed(HERE / "graph_c2s.npz", x=x, knn=32, sigma=8.0,
                        **graph_case(sp, x, 32, 8.0))

    # ---- spmv fixtures --------------------------------------------------
    cases = {}
    for t in range(6):
        n = int(rng.integers(1, 300))
        nnz = int(rng.integers(0, min(n * n, 4000) + 1))
        flat = rng.choice(n * n, size=nnz, replace=False)
        coo = sp.coo_canonicalize(sp.CooMatrix(n, n, flat // n, flat % n,
                                               rng.standard_normal(nnz)))
        csr = sp.coo_to_csr(coo)
        xv = rng.standard_normal(n)
        cases[f"c{t}_row_ptr"] = csr.row_ptr
        cases[f"c{t}_col"] = csr.col_idx
        cases[f"c{t}_vals"] = csr.vals
        cases[f"c{t}_x"] = xv
        cases[f"c{t}_y"] = sp.spmv(csr, xv)
    np.savez_compressed(HERE / "spmv_cases.npz", ncases=6, **cases)

    # ---- eigensolver fixtures -------------------------------------------
    eig = {}
    for t, (n, dens, k) in enumerate([(50, 0.1, 5), (120, 0.05, 8), (300, 0.03, 12)]):
        a = np.zeros((n, n))
        nz = max(1, int(dens * n * n / 2))
        i = rng.integers(0, n, nz)
        j = rng.integers(0, n, nz)
        a[i, j] = rng.standard_normal(nz)
        a = a + a.T
        r, c = np.nonzero(a)
        csr = sp.coo_to_csr(sp.coo_canonicalize(sp.CooMatrix(n, n, r, c, a[r, c])))
        b = sp.eigensolve(csr, sp.LanczosConfig(k=k, seed=0))
        eig[f"e{t}_row_ptr"] = csr.row_ptr
        eig[f"e{t}_col"] = csr.col_idx
        eig[f"e{t}_vals"] = csr.vals
        eig[f"e{t}_k"] = k
        eig[f"e{t}_values"] = b.values
        eig[f"e{t}_vectors"] = b.vectors
        eig[f"e{t}_residuals"] = b.residuals
    np.savez_compressed(HERE / "eigen_cases.npz", ncases=3, **eig)

    # ---- k-means fixtures -----------------------------------------------
    km = {}
    for t, (n, d, k) in enumerate([(400, 5, 7), (1500, 20, 20), (50, 3, 9)]):
        v = rng.standard_normal((n, d)) + 3.0 * rng.standard_normal((k, d))[rng.integers(0, k, n)]
        init_c = sp.kmeanspp_init(v, k, seed=t)
        lab = sp.lloyd(v, init_c, sp.KmeansConfig(k=k))
        full = sp.kmeans(v, sp.KmeansConfig(k=k, seed=t, restarts=2))
        km[f"k{t}_v"] = v
        km[f"k{t}_k"] = k
        km[f"k{t}_chosen"] = chosen_rows(v, init_c)
        km[f"k{t}_labels"] = lab.labels
        km[f"k{t}_centroids"] = lab.centroids
        km[f"k{t}_sse_history"] = lab.sse_history
        km[f"k{t}_iters"] = lab.iters_run
        km[f"k{t}_full_labels"] = full.labels
        km[f"k{t}_full_sse"] = full.sse
        km[f"k{t}_dist"] = sp.pairwise_sq_dist(v[:64], init_c)
    # empty-cluster reseed case (kmeans.py:149-155): duplicate init centroid
    v = np.array([[0.0, 0.0], [0.1, 0.0], [10.0, 0.0], [10.1, 0.0], [50.0, 0.0]])
    init_c = np.array([[0.0, 0.0], [0.0, 0.0], [10.0, 0.0]])
    lab = sp.lloyd(v, init_c, sp.KmeansConfig(k=3))
    km.update(r_v=v, r_init=init_c, r_labels=lab.labels, r_centroids=lab.centroids,
              r_sse_history=lab.sse_history)
    np.savez_compressed(HERE / "kmeans_cases.npz", ncases=3, **km)

    # ---- end-to-end, scaled config 1 (N=2000) -----------------------------
    x, truth = blobs(2000, 32, 20, 1.0, seed=0)
    out = pipeline_case(sp, x, 16, np.sqrt(32.0), 20)
    np.savez_compressed(HERE / "pipeline_c1s.npz", x=x, truth=truth, knn=16,
                        sigma=np.sqrt(32.0), k=20, **out)
    print("small fixtures written", flush=True)

    if args.c1:
        x, truth = blobs(20000, 32, 20, 1.0, seed=0)
        out = pipeline_case(sp, x, 16, np.sqrt(32.0), 20)
        big = {}
        for key in ("row_ptr", "col", "vals", "sym_vals", "edges", "vectors", "embedding"):
            big[key + "_sha"] = sha(out.pop(key))
        out.pop("centroids")
        np.savez_compressed(HERE / "pipeline_c1.npz", truth=truth, knn=16,
                            sigma=np.sqrt(32.0), k=20, n=20000, d=32, **out, **big)
        print("config-1 fixture written", {k: v for k, v in out.items() if k.startswith("t_")})


if __name__ == "__main__":
    main()
