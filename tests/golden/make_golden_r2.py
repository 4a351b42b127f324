"""Round-2 golden vectors for the larger BASELINE.json shapes, made by the
REAL reference package (build container only; the reference tree is not on
the GPU box).

    python tests/golden/make_golden_r2.py --case c3s   # C3 shape, k kept (~8 min)
    python tests/golden/make_golden_r2.py --case c4s   # C4 shape: SBM MatrixInput
    python tests/golden/make_golden_r2.py --case c5s   # C5 shape: Lloyd d=256, k=1000
    python tests/golden/make_golden_r2.py --case c3k   # Lloyd at d=k=1000 (C3's assignment)
    python tests/golden/make_golden_r2.py --case h3    # 20 components (repeated eigenvalue)
    python tests/golden/make_golden_r2.py --case c1p   # config 1 subspace sketch (~2 min)

Inputs that can be regenerated from a seed (blobs, synthetic embeddings) are
not stored; the tests rebuild them and check a SHA-256 of the bytes first.
Eigenvector subspaces of n x k are too large to commit, so each case stores a
projector sketch ``psketch = U_ref (U_ref^T G)`` with G = standard normal
(n x 16) drawn from ``default_rng(SKETCH_SEED)``: for orthonormal U, U_ref,
E |(U U^T - U_ref U_ref^T) G|_F^2 = 16 |U U^T - U_ref U_ref^T|_F^2, and the
Frobenius norm bounds sin of the largest principal angle (tests/test_gpu_shapes.py).

Reference call sites followed: graph.py:185-237, sparse.py:182-187,
laplacian.py:27-106, eigen.py:291-302, pipeline.py:181-267, kmeans.py:107-222,
sbm.py:68-108.
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
SKETCH_SEED = 777
SKETCH_P = 16


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


def embedding_blobs(n, d, k, noise, seed):
    """C5-style synthetic embedding: k Gaussian centres N(0,1) in d dims plus
    N(0, noise^2), rows normalised."""
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, d))
    y = rng.integers(0, k, n)
    v = centers[y] + noise * rng.standard_normal((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return np.ascontiguousarray(v), y


def psketch(u):
    g = np.random.default_rng(SKETCH_SEED).standard_normal((u.shape[0], SKETCH_P))
    return u @ (u.T @ g)


def chosen_rows(v, init_c):
    lut = {v[i].tobytes(): i for i in range(v.shape[0])}
    return np.array([lut[r.tobytes()] for r in init_c], dtype=np.int64)


def spectral(sp, w, k, m=None):
    """degrees -> sym_scale -> eigensolve -> embedding -> k-means++ -> Lloyd,
    exactly the stage calls of pipeline.run (pipeline.py:219-245)."""
    out = {}
    t = {}
    t0 = time.perf_counter()
    d = sp.degrees(w)
    a = sp.sym_scale(w, d)
    t["degrees"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    basis = sp.eigensolve(a, sp.LanczosConfig(k=k, seed=0) if m is None else sp.LanczosConfig(k=k, m=m, seed=0))
    t["eigen"] = time.perf_counter() - t0
    emb = sp.recover_row_eigvecs(basis.vectors, d)
    norms = np.linalg.norm(emb, axis=1, keepdims=True)
    norms[norms == 0.0] = 1.0
    rows = emb / norms
    t0 = time.perf_counter()
    init_c = sp.kmeanspp_init(rows, k, 0)
    t["kmeanspp"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    lab = sp.lloyd(rows, init_c, sp.KmeansConfig(k=k))
    t["lloyd"] = time.perf_counter() - t0
    out.update(degrees_sha=sha(d), values=basis.values, residuals=basis.residuals,
               psketch=psketch(basis.vectors), emb_psketch=psketch(np.linalg.qr(rows)[0]),
               chosen=chosen_rows(rows, init_c), labels=lab.labels.astype(np.int32),
               sse_history=lab.sse_history, iters=lab.iters_run, sse=lab.sse,
               emb_row_sums=rows.sum(axis=1), emb_sq=np.einsum("ij,ij->i", rows, rows),
               )
    for key, val in t.items():
        out["t_" + key] = val
    return out


def case_points(sp, name, n, d, knn, k, cs, m=None, seed=0):
    x, truth = blobs(n, d, k if name != "h3" else 20, cs, seed=seed)
    sigma = float(np.sqrt(d))
    meas = sp.SimilarityMeasure.exp_decay(sigma)
    t0 = time.perf_counter()
    e = sp.build_edges_knn(x, knn, meas)
    w = sp.coo_to_csr(sp.build_similarity(x, e, meas))
    tg = time.perf_counter() - t0
    assert sys.modules["speclust_ref.sparse"].is_symmetric(w)
    out = spectral(sp, w, k, m)
    out.update(x_sha=sha(x), truth=truth.astype(np.int32), n=n, d=d, knn=knn, k=k, cs=cs, seed=seed,
               sigma=sigma, row_ptr_sha=sha(w.row_ptr), col_sha=sha(w.col_idx), vals_sha=sha(w.vals),
               nnz=w.nnz, t_graph=tg, vals_sample=w.vals[:: max(1, w.nnz // 4096)].copy())
    return out


def case_c4s(sp):
    # C4 shape: planted partition with C4's mean degree (~64: ~51 inside the
    # block, ~13 across), unit weights, MatrixInput path (pipeline.py:183-188)
    blocks, size = 100, 100
    cfg = sp.SbmConfig((size,) * blocks, 0.5, 13.0 / (blocks * size - size), seed=4)
    adj, truth = sp.sbm_generate(cfg)
    w = sp.coo_to_csr(adj)
    out = spectral(sp, w, blocks)
    out.update(row_ptr=w.row_ptr, col=w.col_idx.astype(np.int32), truth=truth.astype(np.int32),
               n=w.n_rows, k=blocks)
    return out


def case_lloyd(sp, n, d, k, noise, seed, max_iters):
    v, truth = embedding_blobs(n, d, k, noise, seed)
    idx = np.random.default_rng(0).choice(n, size=k, replace=False)   # kmeans.py:203-205
    t0 = time.perf_counter()
    lab = sp.lloyd(v, v[idx].copy(), sp.KmeansConfig(k=k, max_iters=max_iters))
    t = time.perf_counter() - t0
    return dict(v_sha=sha(v), n=n, d=d, k=k, noise=noise, seed=seed, max_iters=max_iters, init_idx=idx,
                labels=lab.labels.astype(np.int32), centroids_sha=sha(lab.centroids),
                centroids_head=lab.centroids[:8].copy(), sse_history=lab.sse_history,
                iters=lab.iters_run, t_lloyd=t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True, choices=["c3s", "c4s", "c5s", "c3k", "h3", "c1p"])
    a = ap.parse_args()
    sp = load_reference()
    t0 = time.perf_counter()
    if a.case == "c3s":
        out = case_points(sp, "c3s", 20_000, 128, 32, 1000, 1.0)
    elif a.case == "h3":
        out = case_points(sp, "h3", 5000, 32, 16, 20, 3.0)
    elif a.case == "c4s":
        out = case_c4s(sp)
    elif a.case == "c1p":
        # config 1 (N=20k, d=32, kNN=16, k=20): eigenvector subspace sketch for
        # the full-size C1 parity test (pipeline_c1.npz stores digests only)
        x, _ = blobs(20_000, 32, 20, 1.0, seed=0)
        meas = sp.SimilarityMeasure.exp_decay(float(np.sqrt(32.0)))
        w = sp.coo_to_csr(sp.build_similarity(x, sp.build_edges_knn(x, 16, meas), meas))
        d = sp.degrees(w)
        basis = sp.eigensolve(sp.sym_scale(w, d), sp.LanczosConfig(k=20, seed=0))
        out = dict(values=basis.values, psketch=psketch(basis.vectors), x_sha=sha(x))
    elif a.case == "c5s":
        out = case_lloyd(sp, 20_000, 256, 1000, 0.3, 5, 20)
    else:
        out = case_lloyd(sp, 20_000, 1000, 1000, 0.3, 6, 20)
    np.savez_compressed(HERE / f"shape_{a.case}.npz", **out)
    print(a.case, "written in", round(time.perf_counter() - t0, 1), "s",
          {k: v for k, v in out.items() if k.startswith("t_") or k in ("iters", "nnz")}, flush=True)


if __name__ == "__main__":
    main()
