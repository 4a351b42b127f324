"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py).  CPU-only."""

import hashlib

import numpy as np
import pytest

from oracle import speclust_oracle as orc


def _csr_of(g):
    x = g["x"]
    e = orc.knn_edges(x, int(g["knn"]), float(g["sigma"]))
    w = orc.edge_weights(x, e, float(g["sigma"]))
    return e, orc.csr_from_edges(x.shape[0], e, w)


@pytest.mark.parametrize("name", ["graph_blobs600", "graph_underflow", "graph_ties", "graph_c2s"])
def test_graph_bit_exact(golden, name):
    g = golden(name)
    e, (row_ptr, col, vals) = _csr_of(g)
    assert np.array_equal(e, g["edges"])
    assert np.array_equal(row_ptr, g["row_ptr"])
    assert np.array_equal(col, g["col"])
    assert np.array_equal(vals, g["vals"])
    d = orc.degrees(row_ptr, col, vals)
    assert np.array_equal(d, g["degrees"])
    if len(g["sym_vals"]):
        assert np.array_equal(orc.sym_scale_vals(row_ptr, col, vals, d), g["sym_vals"])


def test_spmv_bit_exact(golden):
    g = golden("spmv_cases")
    for t in range(int(g["ncases"])):
        y = orc.spmv_seq(g[f"c{t}_row_ptr"], g[f"c{t}_col"], g[f"c{t}_vals"], g[f"c{t}_x"])
        assert np.array_equal(y, g[f"c{t}_y"])


def test_lanczos_matches_reference(golden):
    g = golden("eigen_cases")
    for t in range(int(g["ncases"])):
        rp, col, vals = g[f"e{t}_row_ptr"], g[f"e{t}_col"], g[f"e{t}_vals"]
        n = len(rp) - 1
        k = int(g[f"e{t}_k"])
        vals_, vecs, res, _ = orc.lanczos_topk(lambda z: orc.spmv_seq(rp, col, vals, z), n, k)
        assert np.array_equal(vals_, g[f"e{t}_values"])
        assert np.array_equal(vecs, g[f"e{t}_vectors"])
        assert np.array_equal(res, g[f"e{t}_residuals"])


def test_kmeans_matches_reference(golden):
    g = golden("kmeans_cases")
    for t in range(int(g["ncases"])):
        v, k = g[f"k{t}_v"], int(g[f"k{t}_k"])
        chosen = orc.kmeanspp_indices(v, k, t)
        assert np.array_equal(chosen, g[f"k{t}_chosen"])
        labels, cent, sse, iters, hist = orc.lloyd(v, v[chosen])
        assert np.array_equal(labels, g[f"k{t}_labels"])
        assert np.array_equal(cent, g[f"k{t}_centroids"])
        assert np.array_equal(hist, g[f"k{t}_sse_history"])
        assert iters == int(g[f"k{t}_iters"])
        full = orc.kmeans(v, k, seed=t, restarts=2)
        assert np.array_equal(full[0], g[f"k{t}_full_labels"])
        assert full[2] == float(g[f"k{t}_full_sse"])
        assert np.array_equal(orc.pairwise_sq_dist(v[:64], v[chosen]), g[f"k{t}_dist"])
    labels, cent, _, _, hist = orc.lloyd(g["r_v"], g["r_init"])
    assert np.array_equal(labels, g["r_labels"])
    assert np.array_equal(cent, g["r_centroids"])
    assert np.array_equal(hist, g["r_sse_history"])


def test_pipeline_scaled_c1(golden):
    g = golden("pipeline_c1s")
    out = orc.run_points(g["x"], int(g["knn"]), float(g["sigma"]), int(g["k"]))
    for key in ("row_ptr", "col", "vals", "degrees", "values", "vectors", "residuals",
                "embedding", "chosen", "labels", "centroids", "sse_history"):
        assert np.array_equal(out[key], g[key]), key
    assert out["ncut"] == float(g["ncut"])
    assert out["iters"] == int(g["iters"])


def test_ari_hand_values():
    assert orc.ari([0, 0, 1, 1], [1, 1, 0, 0]) == 1.0
    assert orc.ari([], []) == 1.0
    assert orc.ari([0, 0, 1, 1], [0, 1, 0, 1]) < 0.0


def test_f_rows_oracle_bit_exact(golden):
    """Oracle restatements of the §8(f) rows (F3 patterns / measures, F4
    metrics and input cleaning) against the real reference (make_golden_f.py)."""
    f = golden("f_rows")
    g = golden("graph_blobs600")
    rp, col, vals = g["row_ptr"], g["col"], g["vals"]
    lab = f["m_labels"]
    assert orc.cut(rp, col, vals, lab) == f["m_cut"]
    assert orc.ratio_cut(rp, col, vals, lab, 6) == f["m_ratio"]
    assert orc.ncut(rp, col, vals, lab) == f["m_ncut"]
    d = orc.degrees(rp, col, vals)
    assert np.array_equal(orc.row_scale_vals(rp, vals, d), f["rs_vals"])
    irp, icol, ivals = f["iso_row_ptr"], f["iso_col"], f["iso_vals"]
    srp, scol, svals, sd, remap = orc.remove_isolated(irp, icol, ivals, orc.degrees(irp, icol, ivals))
    assert np.array_equal(srp, f["iso_sub_row_ptr"]) and np.array_equal(scol, f["iso_sub_col"])
    assert np.array_equal(svals, f["iso_sub_vals"]) and np.array_equal(sd, f["iso_sub_d"])
    assert np.array_equal(remap, f["iso_remap"])
    e = g["edges"]
    for kind in ("cosine", "cross_correlation"):
        for pol in ("clamp_zero", "abs", "keep"):
            v = orc.edge_similarity(g["x"], e, kind, pol)
            want = f[f"sim_{kind}_{pol}_vals"]
            # the reference emits the mirrored COO in canonical (row, col) order
            rows = np.concatenate((e[:, 0], e[:, 1]))
            cols = np.concatenate((e[:, 1], e[:, 0]))
            order = np.lexsort((cols, rows))
            assert np.array_equal(np.concatenate((v, v))[order], want)
    v = orc.edge_similarity(f["sgn_x"], f["sgn_edges"], "cosine", "keep")
    es = f["sgn_edges"]
    order = np.lexsort((np.concatenate((es[:, 1], es[:, 0])), np.concatenate((es[:, 0], es[:, 1]))))
    assert np.array_equal(np.concatenate((v, v))[order], f["sgn_vals"])
    assert np.array_equal(orc.eps_edges(f["eps_x"], float(f["eps_eps"])), f["eps_edges"])
    assert np.array_equal(orc.eps_edges(f["epsd_x"], float(f["epsd_eps"])), f["epsd_edges"])
    assert np.array_equal(orc.threshold_edges_exp(f["thr_x"], float(f["thr_lam"]), float(f["thr_sigma"])),
                          f["thr_edges"])
