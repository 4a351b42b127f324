"""GPU parity of the sharded path's per-shard building blocks (CudaOps -> C ABI)
against the numpy ops / oracle, and of the sharded drivers at world size 1
on CUDA (the NCCL collectives are identity there; their logic is covered
by tests/test_distributed_gloo.py)."""

import numpy as np
import pytest
import torch

from oracle import speclust_oracle as orc
from tests import dist_workers as dw
from tests.np_ops import NumpyOps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_1802_04450_b200.distributed import CudaOps

    return CudaOps()


def cu(a, dtype=torch.float64):
    return torch.from_numpy(np.array(a, copy=True)).to("cuda", dtype)


def test_gemv_blocks(ops):
    rng = np.random.default_rng(0)
    for nl, ld, cnt in [(1, 1, 1), (37, 40, 5), (5000, 5024, 33), (70001, 70016, 130)]:
        B = rng.standard_normal((cnt + 1, ld))
        w = rng.standard_normal(nl)
        h = ops.host(ops.gemv_t(cu(B), cnt, cu(w)))
        want = B[:cnt, :nl] @ w
        assert np.allclose(h, want, rtol=1e-12, atol=1e-12 * np.abs(B[:cnt, :nl]).sum(1).max() * np.abs(w).max())
        wd = cu(w)
        hh = rng.standard_normal(cnt)
        sq = ops.gemv_n(cu(B), cnt, cu(hh), wd, want_sq=True)
        ref = w - B[:cnt, :nl].T @ hh
        assert np.allclose(ops.host(wd), ref, rtol=1e-12, atol=1e-11)
        assert abs(float(sq[0].item()) - ref @ ref) <= 1e-11 * (ref @ ref)


def test_div_and_normal_shard_independent(ops):
    full = ops.host(ops.normal(1000, 0, 42, 3))
    part = ops.host(ops.normal(300, 500, 42, 3))
    assert np.array_equal(full[500:800], part)
    assert abs(full.mean()) < 0.15 and abs(full.std() - 1) < 0.1
    dst = ops.zeros((10,))
    ops.div_into(dst, cu(np.arange(10.0)), 4.0)
    assert np.array_equal(ops.host(dst), np.arange(10.0) / 4.0)


@pytest.mark.parametrize("m,k", [(2, 1), (9, 3), (40, 10), (200, 100), (1000, 20), (2000, 40)])
def test_symeig_block(ops, m, k):
    rng = np.random.default_rng(m)
    T = rng.standard_normal((m, m))
    T = T + T.T
    theta, S = ops.symeig(T, k)
    want = np.sort(np.linalg.eigvalsh(T))[::-1]
    assert np.allclose(theta, want, atol=1e-11 * np.abs(want).max())
    s = ops.host(S)  # (k, m) rows = eigenvectors
    assert np.abs(s @ T @ s.T - np.diag(theta[:k])).max() <= 1e-10 * np.abs(want).max()
    assert np.abs(s @ s.T - np.eye(k)).max() <= 1e-12


def test_ritz_both_layouts(ops):
    rng = np.random.default_rng(1)
    m, k, nl, ld = 30, 7, 1234, 1248
    B = rng.standard_normal((m + 1, ld))
    S = rng.standard_normal((k, m))
    want = S @ B[:m, :nl]
    cm = ops.host(ops.ritz(cu(B), nl, m, cu(S), k))[:, :nl]
    rm = ops.host(ops.ritz(cu(B), nl, m, cu(S), k, rowmajor=True))
    assert np.allclose(cm, want, rtol=1e-12, atol=1e-12)
    assert np.allclose(rm, want.T, rtol=1e-12, atol=1e-12)


def test_embed_blocks(ops):
    rng = np.random.default_rng(2)
    U = rng.standard_normal((501, 6))
    d = rng.uniform(0.5, 3.0, 501)
    V, colsq = ops.embed_scale(cu(U), cu(d))
    Vn, cn = NumpyOps().embed_scale(torch.from_numpy(U), torch.from_numpy(d))
    assert np.allclose(ops.host(V), Vn.numpy(), rtol=1e-15, atol=0)
    assert np.allclose(ops.host(colsq), cn.numpy(), rtol=1e-13)
    for norm in (False, True):
        got = ops.host(ops.embed_finish(V.clone(), colsq, norm))
        want = NumpyOps().embed_finish(Vn.clone(), cn, norm).numpy()
        assert np.allclose(got, want, rtol=1e-13, atol=1e-15)


def test_kmeans_blocks(ops):
    rng = np.random.default_rng(3)
    V = rng.standard_normal((3000, 5))
    C = rng.standard_normal((9, 5))
    np_ops = NumpyOps()
    lab, cost, chg, sse = ops.kmeans_assign(cu(V), cu(C), None)
    lab_n, cost_n, _, sse_n = np_ops.kmeans_assign(torch.from_numpy(V), torch.from_numpy(C), None)
    assert np.array_equal(ops.host(lab), lab_n.numpy())
    assert np.allclose(ops.host(cost), cost_n.numpy(), rtol=1e-12, atol=1e-14)
    assert abs(sse - sse_n) <= 1e-11 * sse_n
    old = lab.clone()
    old[:17] = (old[:17] + 1) % 9
    _, _, chg, _ = ops.kmeans_assign(cu(V), cu(C), old)
    assert chg == 17
    sums, counts = ops.local_sums(cu(V), lab, 12)
    sn, cn = np_ops.local_sums(torch.from_numpy(V), lab_n, 12)
    assert np.array_equal(ops.host(counts), cn.numpy())
    assert np.allclose(ops.host(sums), sn.numpy(), rtol=1e-12, atol=1e-12)
    Cd = ops.host(ops.divide(sums, counts))
    assert np.allclose(Cd, np_ops.divide(sn, cn).numpy(), rtol=1e-12, atol=1e-12)
    assert np.all(Cd[9:] == 0.0)
    c = rng.standard_normal(5000)
    c[10:20] = c.max() + 1  # ties: stable order
    assert np.array_equal(ops.farthest(cu(c), 13), np_ops.farthest(torch.from_numpy(c), 13))


def test_kpp_session_block(ops):
    rng = np.random.default_rng(4)
    V = rng.standard_normal((2000, 4))
    V[100:110] = V[5]  # duplicates -> zero-distance candidates
    a, b = ops.kpp_session(cu(V)), NumpyOps().kpp_session(torch.from_numpy(V))
    try:
        for g in (5, 77, 1999):
            a.take_row(cu(V[g]), g)
            b.take_row(torch.from_numpy(V[g]), g)
            wa, wb = a.weight(), b.weight()
            assert wa[1:] == wb[1:] and abs(wa[0] - wb[0]) <= 1e-12 * wb[0]
            pa, pb = a.psum(wa[0]), b.psum(wb[0])
            assert abs(pa - pb) <= 1e-12
            for t in (0.0, 0.3, 0.999999, pa * 2):
                assert a.search(t) == b.search(t)
            assert a.nth_free(0) == b.nth_free(0) and a.nth_free(1500) == b.nth_free(1500)
    finally:
        a.close()


def test_shard_graph_blocks(ops):
    from paper_1802_04450_b200.sparse import CsrMatrix

    g = orc  # graph from the oracle, sharded rows
    x, _ = orc.blobs(900, 5, 4, 3.0, seed=5)
    e = g.knn_edges(x, 7, 1.3)
    rp, col, vals = g.csr_from_edges(900, e, g.edge_weights(x, e, 1.3))
    w = CsrMatrix(900, 900, rp, col, vals).device()
    d = g.degrees(rp, col, vals)
    scaled = g.sym_scale_vals(rp, col, vals, d)
    labels = np.random.default_rng(0).integers(0, 6, 900)
    r0, r1 = 300, 611
    loc = ops.slice_rows(w, r0, r1)
    assert np.array_equal(ops.host(ops.degrees(loc)), d[r0:r1])
    got = ops.host(ops.sym_scale_shard(loc, r0, cu(d)).vals)
    assert np.array_equal(got, scaled[rp[r0] : rp[r1]])
    bnd, vol, cnt = ops.ncut_partials(loc, r0, cu(labels, torch.int64), 6)
    host = NumpyOps().from_host_csr(CsrMatrix(900, 900, rp, col, vals))
    nb, nv, nc = NumpyOps().ncut_partials(NumpyOps().slice_rows(host, r0, r1), r0, torch.from_numpy(labels), 6)
    assert np.array_equal(ops.host(cnt), nc.numpy())
    assert np.allclose(ops.host(bnd), nb.numpy(), rtol=1e-13)
    assert np.allclose(ops.host(vol), nv.numpy(), rtol=1e-13)


def test_lanczos_sharded_world1_cuda(ops):
    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200.distributed import Comm, lanczos_sharded

    a, m = dw.random_symmetric(n=600, density=0.02, seed=8)
    want = np.sort(np.linalg.eigvalsh(a))[::-1][:6]
    loc = m.device()
    vals, V, res, st = lanczos_sharded(ops, Comm("cuda"), loc, 600, [0, 600], sc.LanczosConfig(k=6, seed=0))
    assert np.max(np.abs(vals - want)) <= 1e-8
    v = ops.host(V)
    assert np.abs(v.T @ v - np.eye(6)).max() <= 1e-8
    assert np.all(res <= 1e-6)


def test_run_sharded_world1_cuda_matches_oracle(ops):
    from paper_1802_04450_b200.distributed import Comm, run_sharded

    x, truth, cfg = dw.blobs_cfg()
    ref = orc.run_points(x, 8, float(np.sqrt(6.0)), 4)
    rep = run_sharded(cfg, Comm("cuda"), ops)
    assert np.max(np.abs(rep.eigenvalues - ref["values"]) / np.abs(ref["values"])) <= 1e-8
    assert orc.ari(rep.labeling.labels, ref["labels"]) >= 0.999
    assert abs(rep.ncut_value - ref["ncut"]) <= 1e-10 * max(1.0, ref["ncut"])


def _assemble(parts):
    rp = [np.zeros(1, dtype=np.int64)]
    off = 0
    for w in parts:
        r = w.row_ptr.cpu().numpy()
        rp.append(r[1:] + off)
        off += int(r[-1])
    col = np.concatenate([w.col.cpu().numpy() for w in parts]).astype(np.int64)
    vals = np.concatenate([w.vals.cpu().numpy() for w in parts])
    return np.concatenate(rp), col, vals


@pytest.mark.parametrize("n,d,knn,world", [(900, 5, 7, 2), (5000, 32, 16, 3), (20000, 64, 32, 5), (300, 4, 3, 4)])
def test_knn_select_union_shards_reassemble(ops, n, d, knn, world):
    """Query-tile shards of the selection + per-rank unions == the one-call
    graph, bit for bit, and == the oracle (graph.py:185-237)."""
    from paper_1802_04450_b200.distributed import row_bounds, scan_bounds
    from paper_1802_04450_b200.graph import knn_graph_device

    import paper_1802_04450_b200 as sc

    x, _ = orc.blobs(n, d, 6, 3.0, seed=n)
    m = sc.SimilarityMeasure.exp_decay(1.7)
    xd = cu(x)
    pb = scan_bounds(n, world)
    sels, perms, svals = [], [], []
    for r in range(world):
        s, p, v = ops.knn_select(xd, knn, m, pb[r], pb[r + 1])
        sels.append(s)
        perms.append(p)
        svals.append(v)
    for p in perms[1:]:
        assert torch.equal(p, perms[0])  # the scan order is replicated
    sel = torch.cat(sels)
    sel_vals = torch.cat(svals)
    rb = row_bounds(n, world)
    full = knn_graph_device(x, knn, m)
    # the value-carrying union (the sharded driver's) and the recomputing one
    for sv in (sel_vals, None):
        parts = [ops.knn_union(xd, knn, m, sel, perms[0], rb[r], rb[r + 1], sv) for r in range(world)]
        rp2, col2, vals2 = _assemble(parts)
        assert np.array_equal(rp2, full.row_ptr.cpu().numpy())
        assert np.array_equal(col2, full.col.cpu().numpy())
        assert np.array_equal(vals2, full.vals.cpu().numpy())
    parts = [ops.knn_union(xd, knn, m, sel, perms[0], rb[r], rb[r + 1], sel_vals) for r in range(world)]
    rp, col, vals = _assemble(parts)
    assert np.array_equal(rp, full.row_ptr.cpu().numpy())
    assert np.array_equal(col, full.col.cpu().numpy())
    assert np.array_equal(vals, full.vals.cpu().numpy())
    if n <= 5000:
        e = orc.knn_edges(x, knn, 1.7)
        orp, ocol, ovals = orc.csr_from_edges(n, e, orc.edge_weights(x, e, 1.7))
        assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
        assert np.all(np.abs(vals - ovals) <= 2 * np.spacing(ovals))  # exp: CUDA vs numpy


def test_knn_union_capacity_error_reports_size(ops):
    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200 import _native as nat
    from paper_1802_04450_b200.errors import BadConfig

    x, _ = orc.blobs(500, 4, 3, 3.0, seed=1)
    m = sc.SimilarityMeasure.exp_decay(1.0)
    xd = cu(x)
    sel, perm, _ = ops.knn_select(xd, 5, m, 0, 500)
    rp = torch.empty(501, dtype=torch.int64, device="cuda")
    col = torch.empty(4, dtype=torch.int32, device="cuda")
    vals = torch.empty(4, dtype=torch.float64, device="cuda")
    nnz = nat.C.c_int64(0)
    rc = nat.load().sc_knn_union_f64(500, 4, nat.ptr(xd), 5, m.two_sigma_sq(), nat.ptr(sel), nat.ptr(perm), 0, 500,
                                     nat.ptr(rp), nat.ptr(col), nat.ptr(vals), 4, nat.C.byref(nnz),
                                     nat.stream_handle())
    assert rc != 0 and nnz.value > 4
    with pytest.raises(BadConfig):
        nat.check(rc)
    w = ops.knn_union(xd, 5, m, sel, perm, 0, 500)
    assert w.nnz == nnz.value
