"""Golden vectors for the SURVEY.md §8(f) rows (F3 patterns / measures, F4
metrics and input cleaning), produced by running the REAL reference package.
Build container only:  python tests/golden/make_golden_f.py  ->  f_rows.npz"""

from __future__ import annotations

import numpy as np

from make_golden import HERE, blobs, load_reference


def main():
    sp = load_reference()
    rng = np.random.default_rng(7_2026)
    out = {}
    g = np.load(HERE / "graph_blobs600.npz")
    w = sp.CsrMatrix(len(g["row_ptr"]) - 1, len(g["row_ptr"]) - 1, g["row_ptr"], g["col"], g["vals"])
    n = w.n_rows
    # ---- F4: cut / ratio_cut / ncut on random 6-part labels
    lab = rng.integers(0, 6, n)
    out.update(m_labels=lab, m_cut=sp.cut(w, lab), m_ratio=sp.ratio_cut(w, lab), m_ncut=sp.ncut(w, lab))
    # ---- F4: row_scale
    d = sp.degrees(w)
    out.update(rs_vals=sp.row_scale(w, d).vals)
    # ---- F4: handle_isolated "remove" on a graph with isolated nodes
    m = 40
    a = (rng.random((m, m)) < 0.15) * rng.random((m, m))
    a = np.triu(a, 1)
    a = a + a.T
    iso = [3, 17, 18, 39]
    a[iso, :] = 0.0
    a[:, iso] = 0.0
    r, c = np.nonzero(a)
    wi = sp.coo_to_csr(sp.coo_canonicalize(sp.CooMatrix(m, m, r, c, a[r, c])))
    di = sp.degrees(wi)
    sub, dsub, remap = sp.handle_isolated(wi, di, "remove")
    out.update(iso_row_ptr=wi.row_ptr, iso_col=wi.col_idx, iso_vals=wi.vals, iso_sub_row_ptr=sub.row_ptr,
               iso_sub_col=sub.col_idx, iso_sub_vals=sub.vals, iso_sub_d=dsub, iso_remap=remap)
    # ---- F3: cosine / cross-correlation edge values over the kNN edges
    x = g["x"]
    e = g["edges"]
    for kind in ("cosine", "cross_correlation"):
        meas = sp.SimilarityMeasure(kind)
        for pol in ("clamp_zero", "abs", "keep"):
            coo = sp.build_similarity(x, e, meas, negative_policy=pol)
            out[f"sim_{kind}_{pol}_rows"] = coo.rows
            out[f"sim_{kind}_{pol}_cols"] = coo.cols
            out[f"sim_{kind}_{pol}_vals"] = coo.vals
    # signed data (cosine values of both signs)
    xs = rng.standard_normal((200, 7))
    es = sp.build_edges_knn(xs, 5, sp.SimilarityMeasure.exp_decay(1.0))
    coo = sp.build_similarity(xs, es, sp.SimilarityMeasure.cosine(), negative_policy="keep")
    out.update(sgn_x=xs, sgn_edges=es, sgn_rows=coo.rows, sgn_cols=coo.cols, sgn_vals=coo.vals)
    # ---- F3: eps pattern
    xe, _ = blobs(700, 5, 7, 3.0, seed=11)
    out.update(eps_x=xe, eps_eps=2.1, eps_edges=sp.build_edges_eps(xe, 2.1))
    # duplicated points: d2 == 0 and exact boundary hits
    xd = np.concatenate((rng.integers(0, 3, (60, 2)).astype(np.float64),) * 2)
    out.update(epsd_x=xd, epsd_eps=1.0, epsd_edges=sp.build_edges_eps(xd, 1.0))
    # ---- F3: threshold pattern (exp_decay)
    out.update(thr_x=xe, thr_sigma=2.0, thr_lam=0.3,
               thr_edges=sp.build_edges_threshold(xe, 0.3, sp.SimilarityMeasure.exp_decay(2.0)))
    # ---- F3 through the pipeline: eps + exp_decay and threshold + cosine
    xp, truth = blobs(400, 6, 4, 4.0, seed=5)
    cfg = sp.PipelineConfig(
        input=sp.PointsInput(measure=sp.SimilarityMeasure.exp_decay(2.0), pattern="eps", points=xp, eps=4.0),
        k_clusters=4, eigen=sp.LanczosConfig(k=4, seed=0), kmeans=sp.KmeansConfig(k=4, seed=0), normalize_rows=True)
    rep = sp.run(cfg)
    out.update(pe_x=xp, pe_truth=truth, pe_labels=rep.labeling.labels, pe_values=rep.eigenvalues, pe_ncut=rep.ncut_value)
    cfg = sp.PipelineConfig(
        input=sp.PointsInput(measure=sp.SimilarityMeasure.cosine(), pattern="threshold", points=xp + 10.0,
                             threshold=0.99),
        k_clusters=4, eigen=sp.LanczosConfig(k=4, seed=0), kmeans=sp.KmeansConfig(k=4, seed=0), normalize_rows=True)
    rep = sp.run(cfg)
    out.update(pt_labels=rep.labeling.labels, pt_values=rep.eigenvalues)
    # ---- F3: kNN pattern with cosine / cross-correlation (n < and >= 4096)
    for tag, (nn, dd, kk, seed) in {"kc1": (600, 8, 10, 21), "kc2": (5000, 16, 12, 22)}.items():
        xk = np.random.default_rng(seed).standard_normal((nn, dd)) + 0.5
        out[f"{tag}_x"] = xk
        out[f"{tag}_knn"] = kk
        for kind in ("cosine", "cross_correlation"):
            meas = sp.SimilarityMeasure(kind)
            ek = sp.build_edges_knn(xk, kk, meas)
            coo = sp.build_similarity(xk, ek, meas, negative_policy="keep")
            out[f"{tag}_{kind}_edges"] = ek
            out[f"{tag}_{kind}_vals"] = coo.vals
    np.savez_compressed(HERE / "f_rows.npz", **out)
    print("f_rows.npz written", {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()
