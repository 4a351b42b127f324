"""One-step lookahead of the device Lanczos drivers (csrc/sc_lanczos.cu,
sc_lanczos::spec_launch / spec_resolve): a common windowed step decides its
couple on the device (the host's cancellation and breakdown tests on the same
doubles) while the next SpMV runs; a declined step falls back to the host
path.  The arithmetic is the same either way, so the solves must be
bit-identical to the ones without lookahead (SPECLUST_LOOKAHEAD=0) -- on a
graph whose sweeps hit exact breakdowns (declines) as well as on a plain one."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(a, k, lookahead, reorth="window"):
    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200.eigen import eigensolve_device

    saved = {v: os.environ.get(v) for v in ("SPECLUST_LOOKAHEAD", "SPECLUST_REORTH")}
    os.environ["SPECLUST_LOOKAHEAD"] = "1" if lookahead else "0"
    os.environ["SPECLUST_REORTH"] = reorth
    try:
        vals, vecs, res, stats = eigensolve_device(a, sc.LanczosConfig(k=k, seed=3))
    finally:
        for v, old in saved.items():
            if old is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = old
    return np.asarray(vals), vecs.cpu().numpy(), np.asarray(res), stats


def _check(a, k):
    v1, u1, r1, s1 = _solve(a, k, True)
    v0, u0, r0, s0 = _solve(a, k, False)
    assert np.array_equal(v1, v0)
    assert np.array_equal(u1, u0)
    assert np.array_equal(r1, r0)
    for key in ("restarts", "matvecs", "breakdowns", "flushes"):
        assert s1[key] == s0[key], key


def test_lookahead_bit_identical_sbm(golden):
    import paper_1802_04450_b200 as sc

    g = golden("shape_c4s")
    n = len(g["row_ptr"]) - 1
    w = sc.CsrMatrix(n, n, g["row_ptr"].astype(np.int64), g["col"].astype(np.int64), np.ones(len(g["col"])))
    a = sc.sym_scale(w, sc.degrees(w)).device()
    for k in (20, 100):
        _check(a, k)


def test_lookahead_bit_identical_breakdowns():
    """Disjoint identical cliques: the operator has two distinct eigenvalues,
    so every Krylov block breaks down exactly after two steps -- the device
    declines those steps and the host's breakdown path (fresh vectors) runs."""
    import paper_1802_04450_b200 as sc

    q, size = 60, 10
    idx = np.arange(q * size).reshape(q, size)
    r = np.repeat(idx, size, axis=1).ravel()
    c = np.tile(idx, (1, size)).ravel()
    m = r != c
    coo = sc.CooMatrix(q * size, q * size, r[m], c[m], np.ones(int(m.sum())))
    w = sc.coo_to_csr(sc.coo_canonicalize(coo))
    a = sc.sym_scale(w, sc.degrees(w)).device()
    v, _, _, s = _solve(a, 12, True)
    assert s["breakdowns"] > 0
    assert np.allclose(v, 1.0)
    _check(a, 12)


def test_lookahead_bit_identical_knn_graph():
    import torch

    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200.graph import knn_graph_device
    from paper_1802_04450_b200.laplacian import degrees_device

    rng = np.random.default_rng(9)
    x = rng.normal(0, 1, (40, 16))[rng.integers(0, 40, 50_000)] + 0.5 * rng.standard_normal((50_000, 16))
    w = knn_graph_device(torch.from_numpy(x).cuda(), 10, sc.SimilarityMeasure.exp_decay(4.0))
    a = sc.sym_scale(w, degrees_device(w))
    _check(a, 40)
