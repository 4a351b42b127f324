"""End-to-end parity of run() on the GPU against the real reference's outputs
(tests/golden/pipeline_c1s.npz: scaled config 1, N=2000; pipeline_c1.npz:
config 1, N=20000, structure stored as SHA-256 digests)."""

import hashlib

import numpy as np
import pytest

import paper_1802_04450_b200 as sc
from oracle import speclust_oracle as orc
from paper_1802_04450_b200.pipeline import run_device

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_for(x, knn, sigma, k):
    return sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(sigma), pattern="knn", points=x, knn=knn),
        k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0),
        normalize_rows=True)


def principal_angle(a, b):
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    s = np.linalg.svd(qa.T @ qb, compute_uv=False)
    return float(np.arccos(np.clip(s.min(), -1.0, 1.0)))


def test_pipeline_scaled_config1(golden):
    g = golden("pipeline_c1s")
    k = int(g["k"])
    rep, wd = run_device(cfg_for(g["x"], int(g["knn"]), float(g["sigma"]), k))
    w = wd.to_host()
    # (1) CSR structure bit-exact, values within a few ulp
    assert np.array_equal(w.row_ptr, g["row_ptr"]) and np.array_equal(w.col_idx, g["col"])
    assert np.max(np.abs(w.vals - g["vals"]) / g["vals"]) < 1e-14
    # (2) eigenvalues (lambda(A) form) 1e-5 relative
    assert np.max(np.abs(rep.eigenvalues - g["values"]) / np.abs(g["values"])) < 1e-5
    assert np.all(rep.eigen_residuals < 1e-6)
    # (3) labels: ARI >= 0.999 vs the reference run
    assert orc.ari(rep.labeling.labels, g["labels"]) >= 0.999
    assert set(rep.timings) == {"graph", "degrees", "eigen", "kmeans", "metrics"}


def test_stage_isolated_kmeans_parity(golden):
    """Same embedding + same init rows -> same labels."""
    g = golden("pipeline_c1s")
    emb = g["embedding"]
    lab = sc.lloyd(emb, emb[g["chosen"]], sc.KmeansConfig(k=int(g["k"])))
    assert orc.ari(lab.labels, g["labels"]) >= 0.999
    assert np.array_equal(sc.kmeanspp_init(emb, int(g["k"]), 0), emb[g["chosen"]])


def test_eigen_subspace_vs_reference(golden):
    g = golden("pipeline_c1s")
    w = sc.CsrMatrix(len(g["degrees"]), len(g["degrees"]), g["row_ptr"], g["col"], g["vals"])
    a = sc.sym_scale(w, g["degrees"])
    b = sc.eigensolve(a, sc.LanczosConfig(k=int(g["k"]), seed=0))
    assert principal_angle(b.vectors, g["vectors"]) < 1e-4


def test_pipeline_config1_full(golden):
    g = golden("pipeline_c1")
    x, truth = orc.blobs(int(g["n"]), int(g["d"]), int(g["k"]), 1.0, seed=0)
    assert np.array_equal(truth, g["truth"])
    k = int(g["k"])
    rep, wd = run_device(cfg_for(x, int(g["knn"]), float(g["sigma"]), k))
    w = wd.to_host()
    assert sha(w.row_ptr) == str(g["row_ptr_sha"])
    assert sha(w.col_idx) == str(g["col_sha"])
    assert np.max(np.abs(rep.eigenvalues - g["values"]) / np.abs(g["values"])) < 1e-5
    assert orc.ari(rep.labeling.labels, g["labels"]) >= 0.999
    # eigenvector subspace vs the reference's (shape_c1p.npz: projector sketch,
    # tests/golden/make_golden_r2.py --case c1p); sin(max angle) <= |P - P_ref|_F
    p = golden("shape_c1p")
    assert np.array_equal(rep.eigenvalues, rep.eigenvalues) and sha(x) == str(p["x_sha"])
    d = sc.degrees(w)
    b = sc.eigensolve(sc.sym_scale(w, d), sc.LanczosConfig(k=k, seed=0))
    gk = np.random.default_rng(777).standard_normal((w.n_rows, 16))
    q, _ = np.linalg.qr(b.vectors)
    dist = np.linalg.norm(q @ (q.T @ gk) - p["psketch"]) / 4.0
    assert dist < 1e-4, dist
    assert np.max(np.abs(b.values - p["values"]) / np.abs(p["values"])) < 1e-5


def test_matrix_input_two_triangles():
    w = np.zeros((6, 6))
    for base in (0, 3):
        for i in range(3):
            for j in range(i + 1, 3):
                w[base + i, base + j] = w[base + j, base + i] = 1.0
    r, c = np.nonzero(w)
    coo = sc.coo_canonicalize(sc.CooMatrix(6, 6, r, c, w[r, c]))
    rep = sc.run(sc.PipelineConfig(input=sc.MatrixInput(matrix=coo), k_clusters=2,
                                   eigen=sc.LanczosConfig(k=2, seed=0), kmeans=sc.KmeansConfig(k=2, seed=0)))
    assert sc.adjusted_rand_index(rep.labeling.labels, [0, 0, 0, 1, 1, 1]) == 1.0
    assert rep.ncut_value == 0.0
    assert np.allclose(rep.eigenvalues, [1.0, 1.0], atol=1e-9)
    assert np.all(rep.eigen_residuals <= 1e-8)


def test_pipeline_errors():
    coo = sc.CooMatrix(3, 3, [0, 1], [1, 0], [1.0, 1.0])
    with pytest.raises(sc.errors.PipelineError) as exc:
        sc.run(sc.PipelineConfig(input=sc.MatrixInput(matrix=coo), k_clusters=2))
    assert exc.value.stage == "degrees"
    assert isinstance(exc.value.cause, sc.errors.IsolatedNode)
    asym = sc.CooMatrix(3, 3, [0, 1, 1, 2], [1, 0, 2, 1], [1.0, 2.0, 1.0, 1.0])
    with pytest.raises(sc.errors.PipelineError) as exc:
        sc.run(sc.PipelineConfig(input=sc.MatrixInput(matrix=asym), k_clusters=2))
    assert exc.value.stage == "graph"
    assert isinstance(exc.value.cause, sc.errors.NotSymmetric)


def test_determinism():
    x, _ = orc.blobs(800, 8, 4, 3.0, seed=7)
    a = sc.run(cfg_for(x, 8, 3.0, 4))
    b = sc.run(cfg_for(x, 8, 3.0, 4))
    assert np.array_equal(a.labeling.labels, b.labeling.labels)
    assert np.array_equal(a.eigenvalues, b.eigenvalues)
    assert a.ncut_value == b.ncut_value


def test_csr_permute_and_gather_rows():
    import torch

    from paper_1802_04450_b200.pipeline import gather_rows_device, permute_device

    rng = np.random.default_rng(3)
    n = 700
    a = (rng.random((n, n)) < 0.02) * rng.standard_normal((n, n))
    # rows of every length class of the kernel: <= 32, 33..64, > 64 entries
    a[:40] += (rng.random((40, n)) < np.linspace(0.03, 0.2, 40)[:, None]) * rng.standard_normal((40, n))
    a = a + a.T
    r, c = np.nonzero(a)
    lens = np.bincount(r, minlength=n)
    assert lens.max() > 64 and np.any((lens > 32) & (lens <= 64)) and np.any(lens <= 32)
    m = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, r, c, a[r, c]))).device()
    perm = rng.permutation(n).astype(np.int32)
    ap, pos = permute_device(m, torch.from_numpy(perm).cuda())
    got = ap.to_host()
    want = a[np.ix_(perm, perm)]
    dense = np.zeros((n, n))
    dense[got.row_indices(), got.col_idx] = got.vals
    assert np.array_equal(dense, want)
    for i in range(n):  # columns strictly increasing per row
        seg = got.col_idx[got.row_ptr[i] : got.row_ptr[i + 1]]
        assert np.all(np.diff(seg) > 0)
    assert np.array_equal(pos.cpu().numpy()[perm], np.arange(n))
    v = torch.from_numpy(rng.standard_normal((n, 5))).cuda()
    g = gather_rows_device(v, pos)
    assert np.array_equal(g.cpu().numpy(), v.cpu().numpy()[pos.cpu().numpy()])


def test_csr_permute_hub_rows():
    """Rows past the warp kernel's shared-memory sort (> 512 entries) go to
    the block kernel: sorted in shared memory up to 8192 entries, counted
    beyond."""
    import scipy.sparse as sps
    import torch

    from paper_1802_04450_b200.pipeline import permute_device

    rng = np.random.default_rng(11)
    n = 12000
    r = rng.integers(0, n, 60000)
    c = rng.integers(0, n, 60000)
    hubs = {0: 9500, 1: 3000, 2: 600, 3: 513}  # row -> number of extra neighbours
    for h, cnt in hubs.items():
        nb = rng.choice(n, cnt, replace=False)
        r = np.concatenate([r, np.full(cnt, h)])
        c = np.concatenate([c, nb])
    a = sps.coo_matrix((rng.standard_normal(len(r)), (r, c)), shape=(n, n)).tocsr()
    a = (a + a.T).tocsr()
    a.sum_duplicates()
    a.sort_indices()
    lens = np.diff(a.indptr)
    assert lens.max() > 8192 and np.any((lens > 512) & (lens <= 8192))
    m = sc.CsrMatrix(n, n, a.indptr.astype(np.int64), a.indices.astype(np.int32), a.data).device()
    perm = rng.permutation(n).astype(np.int32)
    ap, _ = permute_device(m, torch.from_numpy(perm).cuda())
    got = ap.to_host()
    want = a[perm][:, perm].tocsr()
    want.sort_indices()
    assert np.array_equal(got.row_ptr, want.indptr)
    assert np.array_equal(got.col_idx, want.indices)
    assert np.array_equal(got.vals, want.data)


@pytest.mark.parametrize("flag", ["0", "1"])
def test_pipeline_locality_order_eigen(golden, monkeypatch, flag):
    """Eigen stage on P A P^T (kNN locality order) gives the reference's
    spectrum and clustering at C1 (N=20k: a non-trivial scan order)."""
    monkeypatch.setenv("SPECLUST_EIGEN_PERMUTE", flag)
    from paper_1802_04450_b200 import pipeline

    g = golden("pipeline_c1")
    x, _ = orc.blobs(int(g["n"]), int(g["d"]), int(g["k"]), 1.0, seed=0)
    k = int(g["k"])
    rep, wd = pipeline.run_device(cfg_for(x, int(g["knn"]), float(g["sigma"]), k))
    assert pipeline.last_info["eigen"]["locality_order"] == (flag == "1")
    perm = wd.locality_perm.cpu().numpy()
    assert not np.array_equal(perm, np.arange(len(perm)))
    assert np.array_equal(np.sort(perm), np.arange(len(perm)))
    assert np.max(np.abs(rep.eigenvalues - g["values"]) / np.abs(g["values"])) < 1e-5
    assert orc.ari(rep.labeling.labels, g["labels"]) >= 0.999


def test_pipeline_eps_and_threshold_patterns_vs_reference(golden):
    """run() with the eps pattern (exp_decay) and the threshold pattern
    (cosine) -- graph built on the device -- against the real reference's
    run() on the same inputs (tests/golden/f_rows.npz)."""
    f = golden("f_rows")
    x = f["pe_x"]
    cfg = sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(2.0), pattern="eps", points=x, eps=4.0),
        k_clusters=4, eigen=sc.LanczosConfig(k=4, seed=0), kmeans=sc.KmeansConfig(k=4, seed=0), normalize_rows=True)
    rep = sc.run(cfg)
    assert np.max(np.abs(rep.eigenvalues - f["pe_values"])) <= 1e-8
    assert orc.ari(rep.labeling.labels, f["pe_labels"]) >= 0.999
    assert abs(rep.ncut_value - float(f["pe_ncut"])) <= 1e-9 * max(1.0, abs(float(f["pe_ncut"])))
    cfg = sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.cosine(), pattern="threshold", points=x + 10.0,
                             threshold=0.99),
        k_clusters=4, eigen=sc.LanczosConfig(k=4, seed=0), kmeans=sc.KmeansConfig(k=4, seed=0), normalize_rows=True)
    rep = sc.run(cfg)
    assert np.max(np.abs(rep.eigenvalues - f["pt_values"])) <= 1e-8
    assert orc.ari(rep.labeling.labels, f["pt_labels"]) >= 0.999


def test_eigensolve_result_in_basis_matches(monkeypatch):
    """The C4 memory mode (eigenvectors left in the caller-owned Krylov
    basis, embedding built into its unused rows; sc_eigensolve_csr_basis +
    sc_recover_embedding_cm) gives the same eigenpairs, embedding and labels
    as the separate-result path, on an SBM graph (MatrixInput, no locality
    order) and directly at the eigensolver."""
    import torch

    from paper_1802_04450_b200 import _native as nat
    from paper_1802_04450_b200.eigen import eigensolve_device, eigensolve_device_basis
    from paper_1802_04450_b200.laplacian import (degrees_device, recover_embedding_device,
                                                 recover_embedding_from_basis, sym_scale)
    from paper_1802_04450_b200.sbm import SbmConfig, sbm_generate_device

    w, truth = sbm_generate_device(SbmConfig(block_sizes=(400,) * 50, p_in=0.1, p_out=0.002, seed=3))
    k = 50
    cfg = sc.PipelineConfig(input=sc.MatrixInput(matrix=w), k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0),
                            kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
    monkeypatch.setenv("SPECLUST_EIGEN_BASIS", "0")
    ref, _ = run_device(cfg)
    monkeypatch.setenv("SPECLUST_EIGEN_BASIS", "1")
    got, _ = run_device(cfg)
    assert np.array_equal(got.eigenvalues, ref.eigenvalues)
    assert np.allclose(got.eigen_residuals, ref.eigen_residuals, rtol=1e-6, atol=1e-13)
    assert np.array_equal(got.labeling.labels, ref.labeling.labels)
    assert got.labeling.sse == ref.labeling.sse
    # eigensolver level: vectors and the embedding built from the basis rows
    deg = degrees_device(w)
    a = sym_scale(w, deg)
    ecfg = sc.LanczosConfig(k=k, seed=0)
    vals, vecs, res, _ = eigensolve_device(a, ecfg)
    vals_b, basis, ld, res_b, stats = eigensolve_device_basis(a, ecfg)
    n = w.n_rows
    vb = basis[:k, :n].T
    assert np.array_equal(vals, vals_b)
    assert torch.allclose(vb, vecs, rtol=0, atol=1e-12)
    emb = recover_embedding_device(vecs.contiguous(), deg, True)
    emb_b = recover_embedding_from_basis(basis, ld, n, k, deg, True)
    assert emb_b.data_ptr() == basis.data_ptr() + 8 * k * ld  # written into the basis rows k..2k-1
    emb_c = recover_embedding_device(vb.contiguous(), deg, True)
    assert torch.equal(emb_b, emb_c)  # bit-identical to the row-major kernel on the same vectors
    assert torch.allclose(emb_b, emb, rtol=0, atol=1e-11)
    _ = nat


def test_deflated_components_match_plain_solve(monkeypatch):
    """Graphs with 2 <= c < k connected components: the eigenvalue-1 pairs
    locked up front (sc_eigensolve_csr_deflate) + Lanczos on the complement
    give the same eigenvalues, the same eigenvalue-1 eigenspace, residuals
    within tol and the same clustering as the plain solve (the reference's
    procedure, which discovers the copies one verification sweep at a time)."""
    import torch

    from paper_1802_04450_b200 import pipeline as pl

    rng = np.random.default_rng(7)
    nb, per, d = 40, 1000, 12
    centers = rng.normal(0.0, 40.0, (nb, d))
    x = (centers[np.repeat(np.arange(nb), per)] + rng.standard_normal((nb * per, d))).astype(np.float64)
    k = 48
    cfg = cfg_for(x, 10, float(np.sqrt(d)), k)
    monkeypatch.setenv("SPECLUST_DEFLATE", "0")
    ref, _ = run_device(cfg)
    st_ref = dict(pl.last_info["eigen"])
    monkeypatch.setenv("SPECLUST_DEFLATE", "1")
    got, _ = run_device(cfg)
    st = dict(pl.last_info["eigen"])
    assert st["locked"] == nb, st
    assert st["restarts"] <= st_ref["restarts"]
    assert np.abs(got.eigenvalues - ref.eigenvalues).max() <= 1e-9
    assert got.eigen_residuals.max() <= 1e-8
    # k > the 40 planted clusters: k-means splits some of them, and which ones
    # depends on the basis chosen inside the degenerate eigenvalue-1 space
    # (the reference's own choice is arbitrary there too); both clusterings
    # recover the planted partition equally well
    truth = np.repeat(np.arange(nb), per)
    a_got = sc.adjusted_rand_index(got.labeling.labels, truth)
    a_ref = sc.adjusted_rand_index(ref.labeling.labels, truth)
    assert a_got >= 0.9 and a_ref >= 0.9 and abs(a_got - a_ref) <= 0.03, (a_got, a_ref)
    # the eigenvalue-1 eigenspaces agree (the vectors themselves may differ by a rotation inside it)
    from paper_1802_04450_b200.eigen import eigensolve_device, eigensolve_device_deflate
    from paper_1802_04450_b200.graph import knn_graph_device
    from paper_1802_04450_b200.laplacian import degrees_device, sym_scale

    w = knn_graph_device(x, 10, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
    deg = degrees_device(w)
    a = sym_scale(w, deg)
    ecfg = sc.LanczosConfig(k=k, seed=0)
    v0, u0, r0, _ = eigensolve_device(a, ecfg)
    v1, u1, r1, s1 = eigensolve_device_deflate(a, deg, ecfg)
    assert s1["locked"] == nb
    assert np.abs(v1 - v0).max() <= 1e-9
    assert principal_angle(u0[:, :nb].cpu().numpy(), u1[:, :nb].cpu().numpy()) < 1e-6
    assert torch.allclose(u1.T @ u1, torch.eye(k, dtype=torch.float64, device="cuda"), atol=1e-10)
