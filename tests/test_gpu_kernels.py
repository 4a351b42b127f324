"""GPU parity tests of the individual device operators against the golden
vectors of the real reference (tests/golden) and the CPU oracle."""

import numpy as np
import pytest

import paper_1802_04450_b200 as sc
from oracle import speclust_oracle as orc

pytestmark = pytest.mark.gpu


def csr(rp, col, vals):
    n = len(rp) - 1
    return sc.CsrMatrix(n, n, rp, col, vals)


def dense(m):
    out = np.zeros((m.n_rows, m.n_cols))
    out[m.row_indices(), m.col_idx] = m.vals
    return out


# ---------------------------------------------------------------- sparse
def test_spmv_bit_exact_vs_reference(golden):
    g = golden("spmv_cases")
    for t in range(int(g["ncases"])):
        m = csr(g[f"c{t}_row_ptr"], g[f"c{t}_col"], g[f"c{t}_vals"])
        y = sc.spmv(m, g[f"c{t}_x"])
        assert np.array_equal(y, g[f"c{t}_y"]), t


def test_spmv_known_answers():
    eye = sc.coo_to_csr(sc.CooMatrix(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0]))
    assert np.array_equal(sc.spmv(eye, [1.0, 2.0, 3.0]), [1.0, 2.0, 3.0])
    path = sc.coo_to_csr(sc.CooMatrix(3, 3, [0, 1, 1, 2], [1, 0, 2, 1], [1.0] * 4))
    assert np.array_equal(sc.spmv(path, np.ones(3)), [1.0, 2.0, 1.0])
    assert np.array_equal(sc.spmv(path, np.zeros(3)), np.zeros(3))
    with pytest.raises(sc.errors.DimensionMismatch):
        sc.spmv(eye, np.ones(4))
    empty = sc.coo_to_csr(sc.CooMatrix(4, 4, [], [], []))
    assert np.array_equal(sc.spmv(empty, np.ones(4)), np.zeros(4))


def test_spmv_dense_oracle_random():
    rng = np.random.default_rng(11)
    for _ in range(20):
        n = int(rng.integers(1, 200))
        nnz = int(rng.integers(0, min(n * n, 3000) + 1))
        flat = rng.choice(n * n, size=nnz, replace=False)
        m = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, flat // n, flat % n, rng.standard_normal(nnz))))
        x = rng.standard_normal(n)
        want = dense(m) @ x
        got = sc.spmv(m, x)
        assert np.all(np.abs(got - want) <= 1e-12 * max(1.0, np.abs(want).max()))


def test_vectorised_spmv_matches(golden):
    import torch

    from paper_1802_04450_b200 import _native as nat

    g = golden("graph_c2s")
    m = csr(g["row_ptr"], g["col"], g["vals"]).device()
    x = np.random.default_rng(0).standard_normal(m.n_rows)
    xd = torch.from_numpy(x).cuda()
    y = torch.empty_like(xd)
    nat.check(nat.load().sc_spmv_f64(m.n_rows, m.n_cols, nat.ptr(m.row_ptr), nat.ptr(m.col), nat.ptr(m.vals),
                                     nat.ptr(xd), nat.ptr(y), 0, nat.stream_handle()))
    want = orc.spmv_seq(g["row_ptr"], g["col"], g["vals"], x)
    assert np.max(np.abs(y.cpu().numpy() - want)) <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("name", ["graph_blobs600", "graph_ties", "graph_c2s"])
def test_degrees_and_sym_scale_bit_exact(golden, name):
    g = golden(name)
    w = csr(g["row_ptr"], g["col"], g["vals"])
    d = sc.degrees(w)
    assert np.array_equal(d, g["degrees"])
    a = sc.sym_scale(w, d)
    assert np.array_equal(a.vals, g["sym_vals"])


def test_symmetry_gate():
    w = sc.coo_to_csr(sc.CooMatrix(2, 2, [0, 1], [1, 0], [2.0, 2.0]))
    assert sc.sparse.is_symmetric(w)
    a = sc.coo_to_csr(sc.CooMatrix(2, 2, [0], [1], [1.0]))
    assert not sc.sparse.is_symmetric(a)
    b = sc.coo_to_csr(sc.CooMatrix(2, 2, [0, 1], [1, 0], [1.0, 2.0]))
    assert not sc.sparse.is_symmetric(b)
    lower_only = sc.coo_to_csr(sc.CooMatrix(2, 2, [1], [0], [1.0]))
    assert not sc.sparse.is_symmetric(lower_only)
    # random symmetric pattern with a diagonal; then one extra lower entry
    rng = np.random.default_rng(8)
    n = 3000
    r = rng.integers(0, n, 20000)
    c = rng.integers(0, n, 20000)
    v = rng.standard_normal(20000)
    rr = np.concatenate([r, c, np.arange(n)])
    cc = np.concatenate([c, r, np.arange(n)])
    vv = np.concatenate([v, v, np.ones(n)])
    sym = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, rr, cc, vv)))
    assert sc.sparse.is_symmetric(sym)
    keys = set(zip(rr.tolist(), cc.tolist()))
    extra = next((i, j) for i, j in zip(rng.integers(1, n, 100).tolist(), rng.integers(0, n, 100).tolist())
                 if j < i and (i, j) not in keys)
    asym = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, np.append(rr, extra[0]), np.append(cc, extra[1]),
                                                            np.append(vv, 1.0))))
    assert not sc.sparse.is_symmetric(asym)


def test_isolated_and_zero_degree():
    w = sc.coo_to_csr(sc.CooMatrix(4, 4, [0, 1], [1, 0], [1.0, 1.0]))
    d = sc.degrees(w)
    assert np.array_equal(d, [1.0, 1.0, 0.0, 0.0])
    with pytest.raises(sc.errors.IsolatedNode) as exc:
        sc.handle_isolated(w, d)
    assert exc.value.indices == [2, 3]
    sub, dd, remap = sc.handle_isolated(w, d, "remove")
    assert sub.n_rows == 2 and list(remap) == [0, 1, -1, -1]
    with pytest.raises(sc.errors.ZeroDegree):
        sc.sym_scale(w, d)


# ---------------------------------------------------------------- graph
def assert_ulp(got, want, ulps):
    assert got.shape == want.shape
    tol = ulps * np.spacing(np.maximum(np.abs(want), np.finfo(np.float64).tiny))
    assert np.all(np.abs(got - want) <= tol), np.max(np.abs(got - want) / tol) * ulps


def _assert_graph(g, w):
    assert np.array_equal(w.row_ptr, g["row_ptr"])
    assert np.array_equal(w.col_idx, g["col"])
    # values: one exp per pair over d2 summed in numpy's einsum order; d2 is
    # bit-exact, exp is CUDA's vs numpy's (host-SIMD dependent) -> <= 2 ulp
    assert_ulp(w.vals, g["vals"], 2)


@pytest.mark.parametrize("name", ["graph_blobs600", "graph_underflow", "graph_ties", "graph_c2s"])
def test_knn_graph_csr_bit_exact(golden, name):
    from paper_1802_04450_b200.graph import knn_graph_device

    g = golden(name)
    m = sc.SimilarityMeasure.exp_decay(float(g["sigma"]))
    w, stats = knn_graph_device(g["x"], int(g["knn"]), m, return_stats=True)
    _assert_graph(g, w.to_host())
    e = sc.build_edges_knn(g["x"], int(g["knn"]), m)
    assert np.array_equal(e, g["edges"])


def test_knn_small_examples():
    m = sc.SimilarityMeasure.exp_decay(1.0)
    e = sc.build_edges_knn(np.array([[0.0], [1.0], [3.0]]), 1, m)
    assert e.tolist() == [[0, 1], [1, 2]]
    e = sc.build_edges_knn(np.random.default_rng(1).standard_normal((5, 2)), 4, m)
    assert len(e) == 10
    e = sc.build_edges_knn(np.zeros((2, 3)), 1, m)
    assert e.tolist() == [[0, 1]]
    with pytest.raises(ValueError):
        sc.build_edges_knn(np.zeros((3, 1)), 3, m)


@pytest.mark.parametrize("n,d", [(1200, 128), (6000, 256), (20000, 256)])
def test_knn_hub_rows_value_carrying_fill(n, d):
    """A hub point selected by (almost) every other point: its CSR row has far
    more reverse entries than the fill's shared-memory merge holds, so it takes
    the long-row path.  The value-carrying union (exact d2 of each selection
    slot reused) must equal the recomputing union and the oracle."""
    from paper_1802_04450_b200 import _native as nat
    from paper_1802_04450_b200.graph import knn_graph_device, knn_select_device, knn_union_device

    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    x[0] = 0.0  # the hub: at distance 1 from every point, the others ~sqrt(2) apart
    sigma = 0.8
    m = sc.SimilarityMeasure.exp_decay(sigma)
    w = knn_graph_device(x, 2, m).to_host()
    assert np.diff(w.row_ptr)[0] > 256
    if n <= 10000:  # the largest hub (past the shared-memory sort) is checked against the recomputing union
        e = orc.knn_edges(x, 2, sigma)
        want = orc.csr_from_edges(n, e, orc.edge_weights(x, e, sigma))
        assert np.array_equal(w.row_ptr, want[0]) and np.array_equal(w.col_idx, want[1])
        assert_ulp(w.vals, want[2], 2)
    sel, perm = knn_select_device(x, 2, m, 0, n)
    w2 = knn_union_device(x, 2, m, sel, perm, 0, n).to_host()  # recomputes the distances
    assert np.array_equal(w2.col_idx, w.col_idx) and np.array_equal(w2.vals, w.vals)


def test_knn_matches_oracle_random_shapes():
    rng = np.random.default_rng(5)
    for n, d, knn, scale in [(300, 3, 4, 1.0), (513, 17, 9, 0.3), (130, 64, 31, 3.0), (1000, 5, 1, 10.0),
                             (777, 13, 6, 2.0), (2000, 100, 10, 1.0), (1500, 129, 8, 1.0), (1200, 300, 5, 1.0)]:
        x = rng.standard_normal((n, d)) * scale
        sigma = float(np.sqrt(d))
        e = orc.knn_edges(x, knn, sigma)
        want = orc.csr_from_edges(n, e, orc.edge_weights(x, e, sigma))
        m = sc.SimilarityMeasure.exp_decay(sigma)
        from paper_1802_04450_b200.graph import knn_graph_device

        w = knn_graph_device(x, knn, m).to_host()
        assert np.array_equal(w.row_ptr, want[0]), (n, d, knn)
        assert np.array_equal(w.col_idx, want[1]), (n, d, knn)
        assert_ulp(w.vals, want[2], 2)


def test_build_similarity_values(golden):
    g = golden("graph_blobs600")
    m = sc.SimilarityMeasure.exp_decay(float(g["sigma"]))
    coo = sc.build_similarity(g["x"], g["edges"], m)
    w = sc.coo_to_csr(coo)
    _assert_graph(g, w)


# ---------------------------------------------------------------- eigen
def _principal_cos(a, b):
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    return np.linalg.svd(qa.T @ qb, compute_uv=False)


def test_eigensolve_vs_reference(golden):
    g = golden("eigen_cases")
    for t in range(int(g["ncases"])):
        m = csr(g[f"e{t}_row_ptr"], g[f"e{t}_col"], g[f"e{t}_vals"])
        k = int(g[f"e{t}_k"])
        b = sc.eigensolve(m, sc.LanczosConfig(k=k, seed=0))
        ref = g[f"e{t}_values"]
        assert np.max(np.abs(b.values - ref)) <= 1e-8 * max(1.0, np.abs(ref).max())
        assert np.all(b.residuals <= 1e-6 * np.maximum(1.0, np.abs(b.values)))
        defect = np.abs(b.vectors.T @ b.vectors - np.eye(k)).max()
        assert defect <= 1e-8
        cos = _principal_cos(b.vectors, g[f"e{t}_vectors"])
        assert np.min(cos) > np.cos(1e-4)


def test_eigensolve_dense_oracle_and_errors():
    rng = np.random.default_rng(61)
    n = 50
    a = np.zeros((n, n))
    nz = int(0.1 * n * n / 2)
    a[rng.integers(0, n, nz), rng.integers(0, n, nz)] = rng.standard_normal(nz)
    a = a + a.T
    r, c = np.nonzero(a)
    m = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, r, c, a[r, c])))
    want = np.sort(np.linalg.eigvalsh(a))[::-1][:5]
    b = sc.eigensolve(m, sc.LanczosConfig(k=5, seed=0))
    assert np.max(np.abs(b.values - want)) <= 1e-8
    with pytest.raises(ValueError):
        b.values[0] = 1.0
    asym = rng.standard_normal((20, 20))
    r, c = np.nonzero(asym)
    with pytest.raises(sc.errors.NotSymmetric):
        sc.eigensolve(sc.coo_to_csr(sc.CooMatrix(20, 20, r, c, asym[r, c])), sc.LanczosConfig(k=2))
    rect = sc.coo_to_csr(sc.CooMatrix(2, 3, [0, 0, 0, 1, 1, 1], [0, 1, 2, 0, 1, 2], [1.0] * 6))
    with pytest.raises(sc.errors.NotSquare):
        sc.eigensolve(rect, sc.LanczosConfig(k=1, m=2))
    with pytest.raises(sc.errors.MaxRestartsExceeded) as exc:
        big = np.zeros((100, 100))
        nz = 250
        big[rng.integers(0, 100, nz), rng.integers(0, 100, nz)] = rng.standard_normal(nz)
        big = big + big.T
        r, c = np.nonzero(big)
        sc.eigensolve(sc.coo_to_csr(sc.CooMatrix(100, 100, r, c, big[r, c])),
                      sc.LanczosConfig(k=8, m=10, tol=1e-14, max_restarts=0))
    assert exc.value.values is not None and len(exc.value.residuals) == 8


def test_multiplicity_and_disconnected():
    w = sc.coo_to_csr(sc.CooMatrix(4, 4, [0, 1, 2, 3], [1, 0, 3, 2], [1.0] * 4))
    op = sc.sym_scale(w, sc.degrees(w))
    b = sc.eigensolve(op, sc.LanczosConfig(k=2, m=4, seed=0))
    assert np.allclose(b.values, [1.0, 1.0], atol=1e-10)


def drive(s, op):
    while s.state == "need_matvec":
        s.out_slot = op @ s.in_slot
        sc.rci_advance(s)
    return sc.rci_extract(s, lambda v: op @ v)


def test_rci_contract():
    s = sc.rci_new(10, sc.LanczosConfig(k=2, m=6, seed=0))
    assert s.state == "need_matvec"
    assert np.linalg.norm(s.in_slot) == pytest.approx(1.0, abs=1e-14)
    with pytest.raises(sc.errors.NotConverged):
        sc.rci_extract(s, lambda v: v)
    for bad in (dict(k=5, m=5), dict(k=2, m=11), dict(k=2, m=6, tol=0.0)):
        with pytest.raises(sc.errors.BadConfig):
            sc.rci_new(10, sc.LanczosConfig(**bad))
    a = sc.rci_new(16, sc.LanczosConfig(k=2, seed=9))
    b = sc.rci_new(16, sc.LanczosConfig(k=2, seed=9))
    assert np.array_equal(a.in_slot, b.in_slot)


def test_rci_identity_diag_breakdown_path():
    s = sc.rci_new(10, sc.LanczosConfig(k=2, m=6, seed=1))
    basis = drive(s, np.eye(10))
    assert s.restart_count <= 1
    assert np.allclose(basis.values, 1.0, atol=1e-12)
    s = sc.rci_new(9, sc.LanczosConfig(k=2, m=5, seed=3))
    assert np.allclose(drive(s, np.diag(np.arange(9, 0, -1.0))).values, [9.0, 8.0], atol=1e-8)
    s = sc.rci_new(8, sc.LanczosConfig(k=2, m=4, seed=0))
    while s.state == "need_matvec":
        s.out_slot = np.zeros(8)
        sc.rci_advance(s)
    assert s.breakdown_count > 0
    assert np.allclose(sc.rci_extract(s, lambda v: np.zeros(8)).values, 0.0, atol=1e-14)
    w = sc.coo_to_csr(sc.CooMatrix(3, 3, [0, 1, 1, 2], [1, 0, 2, 1], [1.0] * 4))
    op = dense(sc.sym_scale(w, sc.degrees(w)))
    s = sc.rci_new(3, sc.LanczosConfig(k=2, m=3, seed=0))
    assert np.allclose(drive(s, op).values, [1.0, 0.0], atol=1e-8)


def test_rci_rejects_bad_out_slot():
    s = sc.rci_new(6, sc.LanczosConfig(k=2, m=4))
    s.out_slot = np.full(6, np.nan)
    with pytest.raises(sc.errors.BadConfig):
        sc.rci_advance(s)


def test_residual_history_monotone_psd():
    rng = np.random.default_rng(89)
    for trial in range(3):
        b = rng.standard_normal((60, 60)) * (rng.random((60, 60)) < 0.2)
        a = b @ b.T
        s = sc.rci_new(60, sc.LanczosConfig(k=3, m=10, seed=trial))
        while s.state == "need_matvec":
            s.out_slot = a @ s.in_slot
            sc.rci_advance(s)
        hist = s.residual_history
        assert len(hist) >= 1
        for prev, cur in zip(hist, hist[1:]):
            assert cur <= prev * (1.0 + 1e-6) + 1e-12


# ---------------------------------------------------------------- k-means
def test_pairwise_sq_dist():
    s = sc.pairwise_sq_dist(np.array([[0.0, 0.0], [1.0, 0.0]]), np.array([[0.0, 0.0]]))
    assert np.array_equal(s, [[0.0], [1.0]])
    rng = np.random.default_rng(1)
    v = rng.standard_normal((8, 4))
    assert np.array_equal(np.diag(sc.pairwise_sq_dist(v, v)), np.zeros(8))
    v = rng.standard_normal((40, 5))
    c = rng.standard_normal((7, 5))
    naive = ((v[:, None, :] - c[None, :, :]) ** 2).sum(-1)
    assert np.max(np.abs(sc.pairwise_sq_dist(v, c) - naive) / np.maximum(naive, 1e-12)) <= 1e-9
    base = rng.standard_normal((30, 3)) * 1e8
    assert np.all(sc.pairwise_sq_dist(base, base + 1e-9) >= 0.0)
    # the expansion in numpy's einsum order is bit-identical to kmeans.py:84-98
    for n, k, d in [(100, 7, 1), (333, 20, 5), (257, 65, 16), (1000, 100, 100), (200, 13, 137)]:
        v = rng.standard_normal((n, d))
        c = rng.standard_normal((k, d))
        assert np.array_equal(sc.pairwise_sq_dist(v, c), orc.pairwise_sq_dist(v, c)), (n, k, d)
    with pytest.raises(sc.errors.DimensionMismatch):
        sc.pairwise_sq_dist(np.ones((3, 2)), np.ones((2, 3)))


def test_kmeanspp_and_lloyd_vs_reference(golden):
    g = golden("kmeans_cases")
    for t in range(int(g["ncases"])):
        v, k = g[f"k{t}_v"], int(g[f"k{t}_k"])
        init = sc.kmeanspp_init(v, k, t)
        assert np.array_equal(init, v[g[f"k{t}_chosen"]]), t
        lab = sc.lloyd(v, v[g[f"k{t}_chosen"]], sc.KmeansConfig(k=k))
        assert np.array_equal(lab.labels, g[f"k{t}_labels"])
        assert lab.iters_run == int(g[f"k{t}_iters"])
        assert np.allclose(lab.centroids, g[f"k{t}_centroids"], rtol=1e-12, atol=1e-12)
        assert np.allclose(lab.sse_history, g[f"k{t}_sse_history"], rtol=1e-12)
        full = sc.kmeans(v, sc.KmeansConfig(k=k, seed=t, restarts=2))
        assert orc.ari(full.labels, g[f"k{t}_full_labels"]) == 1.0


def test_lloyd_reseed_and_examples(golden):
    g = golden("kmeans_cases")
    lab = sc.lloyd(g["r_v"], g["r_init"], sc.KmeansConfig(k=3))
    assert np.array_equal(lab.labels, g["r_labels"])
    assert np.array_equal(lab.centroids, g["r_centroids"])
    v = np.array([[0.0], [1.0], [10.0], [11.0]])
    lab = sc.lloyd(v, np.array([[0.0], [10.0]]), sc.KmeansConfig(k=2))
    assert lab.labels.tolist() == [0, 0, 1, 1]
    assert np.allclose(lab.centroids.ravel(), [0.5, 10.5])
    lab = sc.lloyd(v, np.array([[3.0]]), sc.KmeansConfig(k=1))
    assert np.allclose(lab.centroids.ravel(), [5.5])
    with pytest.raises(sc.errors.BadConfig):
        sc.kmeans(np.zeros((2, 2)), sc.KmeansConfig(k=3))


def test_ncut_matches_oracle(golden):
    g = golden("graph_blobs600")
    w = csr(g["row_ptr"], g["col"], g["vals"])
    lab = np.random.default_rng(0).integers(0, 6, w.n_rows)
    want = orc.ncut(g["row_ptr"], g["col"], g["vals"], lab)
    assert abs(sc.ncut(w, lab) - want) <= 1e-13 * want
    # pipeline form: empty parts skipped == ncut over np.unique-compacted labels
    from paper_1802_04450_b200.metrics import ncut_device
    import torch

    lab2 = np.where(lab == 3, 5, lab)  # part 3 empty
    val, occ = ncut_device(w.device(), torch.from_numpy(lab2).cuda(), 6, skip_empty=True)
    _, compact = np.unique(lab2, return_inverse=True)
    assert occ == 5
    want2 = orc.ncut(g["row_ptr"], g["col"], g["vals"], compact)
    assert abs(val - want2) <= 1e-13 * want2
    with pytest.raises(sc.errors.ZeroVolumePart):
        sc.ncut(w, lab, k=7)


@pytest.mark.parametrize("fmt", ["sell", "csr"])
def test_eigensolve_spmv_formats(golden, monkeypatch, fmt):
    """The eigensolver's SELL-32-sigma matvec (default for large operators)
    and the CSR one agree with the reference on every eigen golden case."""
    monkeypatch.setenv("SPECLUST_SPMV_FORMAT", fmt)
    g = golden("eigen_cases")
    for t in range(int(g["ncases"])):
        m = csr(g[f"e{t}_row_ptr"], g[f"e{t}_col"], g[f"e{t}_vals"])
        k = int(g[f"e{t}_k"])
        b = sc.eigensolve(m, sc.LanczosConfig(k=k, seed=0))
        ref = g[f"e{t}_values"]
        assert np.max(np.abs(b.values - ref)) <= 1e-8 * max(1.0, np.abs(ref).max())
        assert np.min(_principal_cos(b.vectors, g[f"e{t}_vectors"])) > np.cos(1e-4)


@pytest.mark.parametrize("n_rows,n_cols", [(50_003, 50_003), (1, 7), (300, 300), (20_000, 70_000)])
def test_sell_operator_ragged(n_rows, n_cols):
    """sc_sell_* on ragged rows (empty rows, hub rows far above the mean,
    a row shard with more columns than rows) == the sequential CSR sum up
    to reassociation."""
    import torch

    from paper_1802_04450_b200 import _native as nat

    rng = np.random.default_rng(n_rows)
    deg = rng.integers(0, 90, n_rows)
    deg[rng.random(n_rows) < 0.02] = 0
    hubs = rng.random(n_rows) < 0.003
    deg[hubs] = rng.integers(300, 3000, int(hubs.sum()))
    deg = np.minimum(deg, n_cols)
    rp = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(n_cols, dd, replace=False)) for dd in deg]).astype(np.int64) \
        if deg.sum() else np.zeros(0, np.int64)
    vals = rng.standard_normal(col.size)
    m = sc.CsrMatrix(n_rows, n_cols, rp, col, vals).device()
    x = rng.standard_normal(n_cols)
    want = orc.spmv_seq(rp, col, vals, x)
    lib = nat.load()
    h = nat.vp()
    nat.check(lib.sc_sell_create(n_rows, nat.ptr(m.row_ptr), nat.ptr(m.col), nat.ptr(m.vals), nat.stream_handle(),
                                 nat.C.byref(h)))
    try:
        stored, nlong = nat.C.c_int64(), nat.C.c_int64()
        lib.sc_sell_info(h, nat.C.byref(stored), nat.C.byref(nlong))
        assert nlong.value >= int((deg > max(64, 2 * -(-deg.sum() // n_rows))).sum())
        xd = torch.from_numpy(x).cuda()
        y = torch.full((n_rows,), np.nan, dtype=torch.float64, device="cuda")
        nat.check(lib.sc_sell_spmv(h, nat.ptr(xd), nat.ptr(y), nat.stream_handle()))
        got = y.cpu().numpy()
    finally:
        lib.sc_sell_destroy(h)
    bound = 1e-13 * np.maximum(1.0, orc.spmv_seq(rp, col, np.abs(vals), np.abs(x)))
    assert np.all(np.abs(got - want) <= bound)


def _ragged_csr(n_rows, n_cols, seed):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 90, n_rows)
    deg[rng.random(n_rows) < 0.02] = 0
    hubs = rng.random(n_rows) < 0.003
    deg[hubs] = rng.integers(300, 5000, int(hubs.sum()))
    deg = np.minimum(deg, n_cols)
    rp = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(n_cols, dd, replace=False)) for dd in deg]).astype(np.int64) \
        if deg.sum() else np.zeros(0, np.int64)
    vals = rng.standard_normal(col.size)
    return rp, col, vals, rng.standard_normal(n_cols)


@pytest.mark.parametrize("kernel", ["placed", "local", "vec", "affine", "pipe", "batch2", "batch4", "batch8", "bulk"])
@pytest.mark.parametrize("n_rows,n_cols", [(60_001, 60_001), (5000, 5000), (1, 7), (20_000, 70_000)])
def test_spmv_kernels_and_plan_ragged(monkeypatch, kernel, n_rows, n_cols):
    """Every SpMV kernel variant, through sc_spmv_f64 and through an
    sc_spmv_plan (bulk-staged chunks, hub rows read directly, a ragged tail
    chunk), equals the sequential CSR sum up to reassociation, on rows from
    empty to 5000 nonzeros and on a row shard with more columns than rows."""
    import torch

    from paper_1802_04450_b200 import _native as nat

    monkeypatch.setenv("SPECLUST_SPMV_KERNEL", kernel)
    rp, col, vals, x = _ragged_csr(n_rows, n_cols, n_rows + len(kernel))
    m = sc.CsrMatrix(n_rows, n_cols, rp, col, vals).device()
    want = orc.spmv_seq(rp, col, vals, x)
    bound = 1e-13 * np.maximum(1.0, orc.spmv_seq(rp, col, np.abs(vals), np.abs(x)))
    lib = nat.load()
    xd = torch.from_numpy(x).cuda()
    y = torch.full((n_rows,), np.nan, dtype=torch.float64, device="cuda")
    nat.check(lib.sc_spmv_f64(n_rows, n_cols, nat.ptr(m.row_ptr), nat.ptr(m.col), nat.ptr(m.vals), nat.ptr(xd),
                              nat.ptr(y), 0, nat.stream_handle()))
    assert np.all(np.abs(y.cpu().numpy() - want) <= bound)
    h = nat.vp()
    nat.check(lib.sc_spmv_plan_create(n_rows, nat.ptr(m.row_ptr), nat.ptr(m.col), nat.ptr(m.vals),
                                      nat.stream_handle(), nat.C.byref(h)))
    try:
        for _ in range(2):  # the plan is reusable
            y.fill_(np.nan)
            nat.check(lib.sc_spmv_plan_apply(h, nat.ptr(xd), nat.ptr(y), nat.stream_handle()))
            assert np.all(np.abs(y.cpu().numpy() - want) <= bound)
    finally:
        lib.sc_spmv_plan_destroy(h)


_VARIANT_CASES = []


def _variant_cases():
    """Blobs cases + their oracle CSR, computed once for all variants."""
    if not _VARIANT_CASES:
        rng = np.random.default_rng(17)
        for n, d, knn in [(6000, 32, 16), (5000, 64, 32), (4500, 100, 10)]:
            centers = rng.normal(0.0, 0.7, (12, d))
            x = centers[rng.integers(0, 12, n)] + rng.standard_normal((n, d))
            sigma = float(np.sqrt(d))
            e = orc.knn_edges(x, knn, sigma)
            _VARIANT_CASES.append((x, knn, sigma, orc.csr_from_edges(n, e, orc.edge_weights(x, e, sigma))))
    return _VARIANT_CASES


@pytest.mark.parametrize("variant", [{}, {"SPECLUST_KNN_TC": "1"}, {"SPECLUST_KNN_HEAP": "1"},
                                     {"SPECLUST_KNN_KERNEL": "simt"}, {"SPECLUST_KNN_NOTOUR": "1"}])
def test_knn_kernel_variants_match_oracle(monkeypatch, variant):
    """Every candidate-kernel variant (query-pair tcgen05 kernel with global
    lists or shared heaps, the one-tile tcgen05 kernel, the SIMT kernel, the
    untoured pivot order) yields the reference CSR bit-for-bit on blobs large
    enough for the locality order (n >= 4096), for d = 32, 64 and 100."""
    from paper_1802_04450_b200.graph import knn_graph_device

    for k_, v_ in variant.items():
        monkeypatch.setenv(k_, v_)
    for x, knn, sigma, want in _variant_cases():
        w = knn_graph_device(x, knn, sc.SimilarityMeasure.exp_decay(sigma)).to_host()
        assert np.array_equal(w.row_ptr, want[0]), (x.shape, knn)
        assert np.array_equal(w.col_idx, want[1]), (x.shape, knn)
        assert_ulp(w.vals, want[2], 2)


def _lloyd_cases():
    rng = np.random.default_rng(23)
    out = []
    for n, d, k, kind in [(20_000, 100, 100, "unit"), (9_000, 16, 10, "unit"), (12_000, 200, 300, "unit"),
                          (8_192, 64, 50, "raw"), (6_000, 33, 40, "dup"),
                          # dp > 256: the K-chunk-streaming kernel (odd tile count: a half-full last CTA)
                          (4_200, 300, 130, "unit"), (5_000, 520, 64, "dup"),
                          # d = 256 (two resident point tiles per CTA); three centroids per planted
                          # cluster: many rows sit between two or three centroids (near ties
                          # settled by the kept three candidates, as_resolve_kernel)
                          (10_000, 256, 600, "unit"), (9_000, 192, 240, "split"), (8_500, 256, 300, "split")]:
        nc = k // 3 if kind == "split" else k
        centers = rng.normal(0.0, 1.0, (nc, d))
        v = centers[rng.integers(0, nc, n)] + 0.3 * rng.standard_normal((n, d))
        if kind in ("unit", "split"):
            v /= np.linalg.norm(v, axis=1, keepdims=True)
        elif kind == "raw":
            v *= 1e3  # large magnitudes: exercises the operand scaling
        else:
            v[n // 2:] = v[: n - n // 2]  # exact duplicate rows -> exact ties / zero costs
        init = v[rng.choice(n, k, replace=False)].copy()
        out.append((v, init, k))
    return out


def test_lloyd_tensor_core_assignment_bit_identical(monkeypatch):
    """The tcgen05 assignment with certified argmin (n >= 4096) yields
    labels, centroids, SSE history and iteration counts bit-identical to the
    CPU oracle's restatement of kmeans.py:159-196 (pinned to the reference by
    tests/test_oracle_golden.py) and to the library's fp64 path, on unit-norm
    embeddings, raw large-magnitude data and data with exact duplicate rows."""
    for v, init, k in _lloyd_cases():
        cfg = sc.KmeansConfig(k=k, max_iters=40)
        got = sc.lloyd(v, init, cfg)
        labels, cent, sse, iters, hist = orc.lloyd(v, init, max_iters=40)
        assert got.iters_run == iters, v.shape
        assert np.array_equal(got.labels, labels), v.shape
        assert np.array_equal(got.centroids, cent), v.shape
        assert np.array_equal(got.sse_history, hist), v.shape
        monkeypatch.setenv("SPECLUST_ASSIGN", "fp64")
        ref = sc.lloyd(v, init, cfg)
        monkeypatch.delenv("SPECLUST_ASSIGN")
        assert np.array_equal(got.labels, ref.labels) and np.array_equal(got.sse_history, ref.sse_history)


# ---------------------------------------------------------------- §8(f) rows
def test_f4_metrics_and_cleaning_vs_reference(golden):
    """cut / ratio_cut / ncut, row_scale and handle_isolated('remove') on the
    device against the real reference's outputs (tests/golden/f_rows.npz)."""
    f = golden("f_rows")
    g = golden("graph_blobs600")
    w = csr(g["row_ptr"], g["col"], g["vals"])
    lab = f["m_labels"]
    assert abs(sc.cut(w, lab) - f["m_cut"]) <= 1e-13 * f["m_cut"]
    assert abs(sc.ratio_cut(w, lab) - f["m_ratio"]) <= 1e-13 * f["m_ratio"]
    assert abs(sc.ncut(w, lab) - f["m_ncut"]) <= 1e-13 * f["m_ncut"]
    with pytest.raises(sc.errors.EmptyPart):
        sc.ratio_cut(w, np.where(lab == 2, 1, lab), k=6)
    d = sc.degrees(w)
    assert np.array_equal(sc.row_scale(w, d).vals, f["rs_vals"])  # IEEE division: bit-exact
    wi = csr(f["iso_row_ptr"], f["iso_col"], f["iso_vals"])
    sub, dsub, remap = sc.handle_isolated(wi, sc.degrees(wi), "remove")
    assert np.array_equal(sub.row_ptr, f["iso_sub_row_ptr"]) and np.array_equal(sub.col_idx, f["iso_sub_col"])
    assert np.array_equal(sub.vals, f["iso_sub_vals"]) and np.array_equal(dsub, f["iso_sub_d"])
    assert np.array_equal(remap, f["iso_remap"])


def test_f3_measures_and_patterns_vs_reference(golden):
    """cosine / cross-correlation edge similarities (all negative policies),
    the eps pattern and the exp_decay threshold pattern on the device against
    the real reference (bit-exact); degenerate points raise DegenerateVector."""
    f = golden("f_rows")
    g = golden("graph_blobs600")
    for kind in ("cosine", "cross_correlation"):
        for pol in ("clamp_zero", "abs", "keep"):
            coo = sc.build_similarity(g["x"], g["edges"], sc.SimilarityMeasure(kind), negative_policy=pol)
            assert np.array_equal(coo.rows, f[f"sim_{kind}_{pol}_rows"])
            assert np.array_equal(coo.cols, f[f"sim_{kind}_{pol}_cols"])
            assert np.array_equal(coo.vals, f[f"sim_{kind}_{pol}_vals"]), (kind, pol)
    coo = sc.build_similarity(f["sgn_x"], f["sgn_edges"], sc.SimilarityMeasure.cosine(), negative_policy="keep")
    assert np.array_equal(coo.vals, f["sgn_vals"])
    assert np.array_equal(sc.build_edges_eps(f["eps_x"], float(f["eps_eps"])), f["eps_edges"])
    assert np.array_equal(sc.build_edges_eps(f["epsd_x"], float(f["epsd_eps"])), f["epsd_edges"])
    e = sc.build_edges_threshold(f["thr_x"], float(f["thr_lam"]), sc.SimilarityMeasure.exp_decay(float(f["thr_sigma"])))
    assert np.array_equal(e, f["thr_edges"])
    x = np.random.default_rng(3).standard_normal((50, 4))
    x[7] = 0.0
    with pytest.raises(sc.errors.DegenerateVector) as exc:
        sc.build_similarity(x, [[7, 9], [1, 2]], sc.SimilarityMeasure.cosine())
    assert exc.value.index == 7
    x[11] = 3.0  # constant row: degenerate for cross_correlation only
    sc.build_similarity(x, [[11, 9]], sc.SimilarityMeasure.cosine())
    with pytest.raises(sc.errors.DegenerateVector):
        sc.build_similarity(x, [[11, 9]], sc.SimilarityMeasure.cross_correlation())
    # cosine threshold vs the oracle's cosine values (einsum-order dots)
    xs = f["sgn_x"]
    e = sc.build_edges_threshold(xs, 0.5, sc.SimilarityMeasure.cosine())
    allp = np.array([[i, j] for i in range(len(xs)) for j in range(i + 1, len(xs))])
    v = orc.edge_similarity(xs, allp, "cosine", "keep")
    assert np.array_equal(e, allp[v > 0.5])


@pytest.mark.parametrize("tag", ["kc1", "kc2"])
@pytest.mark.parametrize("kind", ["cosine", "cross_correlation"])
def test_knn_cosine_cross_correlation_vs_reference(golden, tag, kind):
    """kNN pattern with the cosine / cross-correlation measures on the device
    (tensor-core candidates on the row-normalised points, exact ranking by the
    reference's similarity, certificate in cosine space) == the real
    reference's build_edges_knn + build_similarity; kc2 (n = 5000) takes the
    locality-ordered tcgen05 path."""
    f = golden("f_rows")
    x, knn = f[f"{tag}_x"], int(f[f"{tag}_knn"])
    m = sc.SimilarityMeasure(kind)
    e = sc.build_edges_knn(x, knn, m)
    assert np.array_equal(e, f[f"{tag}_{kind}_edges"])
    from paper_1802_04450_b200.graph import knn_graph_device

    w = knn_graph_device(x, knn, m, negative_policy="keep").to_host()
    coo = sc.build_similarity(x, e, m, negative_policy="keep")
    assert np.array_equal(w.vals, coo.vals) and np.array_equal(w.vals, f[f"{tag}_{kind}_vals"])
    assert sc.sparse.is_symmetric(w)


def test_sbm_generator_statistics():
    """Device planted-partition SBM (sc_sbm_csr): canonical symmetric unit
    CSR without self-loops; intra / inter edge counts within 5 sigma of the
    binomial means of the reference's model (sbm.py:68-108); deterministic
    per seed, different across seeds; p = 0 / p = 1 edge cases."""
    cfg = sc.SbmConfig(block_sizes=(700, 500, 800, 650), p_in=0.05, p_out=0.002, seed=3)
    adj, lab = sc.sbm_generate(cfg)
    n = sum(cfg.block_sizes)
    assert adj.n_rows == n and np.array_equal(lab, np.repeat(np.arange(4), cfg.block_sizes))
    assert np.all(adj.vals == 1.0) and not np.any(adj.rows == adj.cols)
    order = np.lexsort((adj.cols, adj.rows))
    assert np.array_equal(order, np.arange(adj.nnz))  # canonical
    key = set(zip(adj.rows.tolist(), adj.cols.tolist()))
    assert all((c, r) in key for r, c in key)  # symmetric
    intra = int(np.sum(lab[adj.rows] == lab[adj.cols])) // 2
    inter = adj.nnz // 2 - intra
    sizes = np.array(cfg.block_sizes)
    n_in = int(np.sum(sizes * (sizes - 1) // 2))
    n_out = n * (n - 1) // 2 - n_in
    for got, pairs, p in ((intra, n_in, cfg.p_in), (inter, n_out, cfg.p_out)):
        mu, sd = pairs * p, np.sqrt(pairs * p * (1 - p))
        assert abs(got - mu) <= 5 * sd, (got, mu, sd)
    adj2, _ = sc.sbm_generate(cfg)
    assert np.array_equal(adj2.rows, adj.rows) and np.array_equal(adj2.cols, adj.cols)
    adj3, _ = sc.sbm_generate(sc.SbmConfig(block_sizes=cfg.block_sizes, p_in=0.05, p_out=0.002, seed=4))
    assert not (adj3.nnz == adj.nnz and np.array_equal(adj3.cols, adj.cols))
    full, _ = sc.sbm_generate(sc.SbmConfig(block_sizes=(5, 4), p_in=1.0, p_out=0.0))
    assert full.nnz == 5 * 4 + 4 * 3
    empty, _ = sc.sbm_generate(sc.SbmConfig(block_sizes=(5, 4), p_in=0.0, p_out=0.0))
    assert empty.nnz == 0


@pytest.mark.parametrize("sizes,p_in,p_out", [((100,) * 200, 0.3, 0.01),   # Syn200 (test_acceptance.py:186)
                                              ((300,), 1.0, 0.0),           # dense: 299 lower neighbours
                                              ((3000,), 1.0, 0.0),          # past the shared-memory bitonic? no: 2999
                                              ((20000,), 1.0, 0.0)])        # rank-counting path (19999 > 16384)
def test_sbm_long_rows(sizes, p_in, p_out):
    """Rows with more than 256 (and more than 16384) lower-triangle
    neighbours: canonical CSR, exact edge count when p = 1."""
    import torch
    from paper_1802_04450_b200.sbm import sbm_generate_device

    w, _ = sbm_generate_device(sc.SbmConfig(block_sizes=sizes, p_in=p_in, p_out=p_out, seed=5))
    rp = w.row_ptr.cpu().numpy()
    col = w.col.cpu().numpy().astype(np.int64)
    n = rp.size - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.all(np.diff(col)[np.diff(rows) == 0] > 0)  # strictly increasing per row
    assert not np.any(col == rows)
    if p_in == 1.0:
        assert w.nnz == n * (n - 1)
    else:
        assert abs(w.nnz / 2 - 2_288_817) < 30_000  # Syn200's edge count in the reference
    # symmetric: the transpose has the same canonical order
    t = np.lexsort((rows, col))
    assert np.array_equal(col[t], rows) and np.array_equal(rows[t], col)
    del torch


def test_sbm_pipeline_and_binary_input(tmp_path):
    """A device-generated SBM clustered through MatrixInput from a binary CSR
    container (F2 path): recovers the planted blocks (ARI >= 0.95, the
    reference's own SBM acceptance bar, test_pipeline.py)."""
    from paper_1802_04450_b200 import io
    from paper_1802_04450_b200.sbm import sbm_generate_device

    w, lab = sbm_generate_device(sc.SbmConfig(block_sizes=(400,) * 10, p_in=0.08, p_out=0.002, seed=1))
    io.save_csr_binary(tmp_path / "g.scb", w)
    rep = sc.run(sc.PipelineConfig(input=sc.MatrixInput(path=str(tmp_path / "g.scb")), k_clusters=10,
                                   eigen=sc.LanczosConfig(k=10, seed=0), kmeans=sc.KmeansConfig(k=10, seed=0),
                                   normalize_rows=True))
    assert sc.adjusted_rand_index(rep.labeling.labels, lab.cpu().numpy()) >= 0.95


def test_kmeanspp_fp16_screen_exact(monkeypatch):
    """k-means++ with the fp16 screen of the D^2 update (d >= 32) and the
    identical-row groups (one distance per group) draws the same rows as the
    CPU oracle's restatement of kmeans.py:107-136 (pinned to the reference by
    tests/test_oracle_golden.py) and as the unscreened update: the screen
    only skips rows whose certified lower bound exceeds their current D^2.
    Unit-norm embeddings, raw large-magnitude data, exact duplicates (zero
    distances, ties) and mostly-one-hot rows (the embedding rows of locked
    graph components)."""
    rng = np.random.default_rng(31)
    for n, d, k, kind in [(20_000, 100, 100, "unit"), (6_000, 300, 40, "raw"), (5_000, 64, 30, "dup"),
                          (30_000, 64, 80, "onehot")]:
        centers = rng.normal(0.0, 1.0, (k, d))
        v = centers[rng.integers(0, k, n)] + 0.2 * rng.standard_normal((n, d))
        if kind == "unit":
            v /= np.linalg.norm(v, axis=1, keepdims=True)
        elif kind == "raw":
            v *= 3e4
        elif kind == "dup":
            v[n // 2:] = v[: n - n // 2]
        else:  # rows of locked components: 60 distinct one-hot rows for 80 % of the points
            hot = np.eye(d)[rng.integers(0, 60, n)]
            v /= np.linalg.norm(v, axis=1, keepdims=True)
            keep = rng.random(n) < 0.8
            v[keep] = hot[keep]
        v = np.ascontiguousarray(v)
        want = orc.kmeanspp_indices(v, k, 7)
        init = sc.kmeanspp_init(v, k, 7)
        assert np.array_equal(init, v[want]), (n, d, kind)
        monkeypatch.setenv("SPECLUST_KPP_SCREEN", "0")
        monkeypatch.setenv("SPECLUST_KPP_DEDUP", "0")
        plain = sc.kmeanspp_init(v, k, 7)
        monkeypatch.delenv("SPECLUST_KPP_SCREEN")
        monkeypatch.delenv("SPECLUST_KPP_DEDUP")
        assert np.array_equal(plain, init)


def test_kmeanspp_zero_panels_exact(monkeypatch):
    """k-means++ on embeddings whose rows are mostly zero 8-column panels
    (C3's embedding: each row has one nonzero among the locked component
    columns plus a dense tail): the update skips loading zero panels and must
    still draw the oracle's rows (kmeans.py:107-136), bit-identically to the
    update with the skip switched off (SPECLUST_KPP_ZERO_PANELS=0)."""
    rng = np.random.default_rng(43)
    for n, d, k, ncomp, dense in [(30_000, 200, 60, 150, 24), (20_000, 77, 40, 60, 5), (12_000, 1000, 50, 850, 150)]:
        comp = rng.integers(0, ncomp, n)
        v = np.zeros((n, d))
        v[np.arange(n), comp] = 1.0 + 0.01 * rng.standard_normal(n)
        v[:, d - dense:] = 0.05 * rng.standard_normal((n, dense))
        v[rng.random(n) < 0.1, d - dense:] = 0.0  # some rows without a dense tail
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        v = np.ascontiguousarray(v)
        want = orc.kmeanspp_indices(v, k, 5)
        init = sc.kmeanspp_init(v, k, 5)
        assert np.array_equal(init, v[want]), (n, d)
        monkeypatch.setenv("SPECLUST_KPP_ZERO_PANELS", "0")
        assert np.array_equal(sc.kmeanspp_init(v, k, 5), init), (n, d)
        monkeypatch.delenv("SPECLUST_KPP_ZERO_PANELS")
