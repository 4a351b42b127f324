"""CPU oracle for the spectral-clustering hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the algorithm of the reference package
``speclust`` (``/root/reference/pkg/src/speclust``) for the path named by
BASELINE.json's north star: kNN + exp_decay similarity graph -> CSR ->
degrees -> symmetric normalisation -> thick-restart Lanczos -> eigenvector
recovery (+ row normalisation) -> k-means++ / Lloyd -> ncut.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
    baseline / ``--impl reference`` arm may import this module.  The product
    package ``paper_1802_04450_b200`` never does; it has no CPU fallback.
  * Every function cites the reference file:line whose semantics it follows.
    Where the reference's numerics are fixed by a numpy primitive (einsum,
    bincount, lexsort, cumsum) the same primitive is used here, so in the
    same numpy build the oracle reproduces the reference bit-for-bit.
  * Pinning: ``tests/golden/make_golden.py`` runs the real reference package
    (importable in the build container only) and stores its outputs under
    ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this oracle
    against every stored vector.

Short forms: ``graph.py:N`` = /root/reference/pkg/src/speclust/graph.py line N.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "blobs",
    "knn_edges",
    "edge_weights",
    "csr_from_edges",
    "spmv_seq",
    "degrees",
    "sym_scale_vals",
    "lanczos_topk",
    "recover_embedding",
    "normalize_rows",
    "pairwise_sq_dist",
    "kmeanspp_indices",
    "lloyd",
    "kmeans",
    "ncut",
    "ari",
    "run_points",
]

BREAKDOWN_RTOL = 1e-13  # eigen.py:50


# --------------------------------------------------------------------------
# synthetic inputs (SURVEY.md §8(d) "Synthetic inputs")
# --------------------------------------------------------------------------
def blobs(n: int, d: int, k: int, center_scale: float, seed: int = 0):
    """Seeded Gaussian blobs: centers ~ N(0, cs^2), labels uniform, unit noise."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, center_scale, (k, d))
    y = rng.integers(0, k, n)
    x = centers[y] + rng.standard_normal((n, d))
    return np.ascontiguousarray(x), y


# --------------------------------------------------------------------------
# stage 1: kNN graph (graph.py:149-157, 185-204, 136-141, 214-237)
# --------------------------------------------------------------------------
def _row_sq_dist(x: np.ndarray, i: int) -> np.ndarray:
    # graph.py:92 (_sq_norms) applied to x - x[i] as in graph.py:156
    diff = x - x[i]
    return np.einsum("ij,ij->i", diff, diff)


def knn_select_row(x: np.ndarray, i: int, knn: int, inv: float) -> np.ndarray:
    """Indices of the ``knn`` most similar points of row i.

    Ranking key (graph.py:198-202): similarity descending, index ascending,
    similarity s = exp(inv * d2) with inv = -1/(2 sigma^2) (graph.py:154-156).
    Instead of a full lexsort the boundary value is found with a partition;
    ties at the boundary are resolved toward lower indices, which is exactly
    what the lexsort key does.
    """
    n = x.shape[0]
    s = np.exp(inv * _row_sq_dist(x, i))
    s[i] = -np.inf  # self excluded (graph.py:197 np.delete)
    neg = -s
    kth = np.partition(neg, knn - 1)[knn - 1]
    strict = np.flatnonzero(neg < kth)
    ties = np.flatnonzero(neg == kth)
    take = knn - len(strict)
    sel = np.concatenate((strict, ties[:take]))
    assert len(sel) == knn and i not in sel
    del n
    return sel


def knn_edges(x, knn: int, sigma: float) -> np.ndarray:
    """Union kNN pattern, pairs (i, j) with i < j in row-major order
    (graph.py:185-204)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    if not 1 <= knn < n:
        raise ValueError("knn must satisfy 1 <= knn < n")
    inv = -1.0 / (2.0 * sigma**2)
    rows = np.repeat(np.arange(n, dtype=np.int64), knn)
    cols = np.empty(n * knn, dtype=np.int64)
    for i in range(n):
        cols[i * knn:(i + 1) * knn] = knn_select_row(x, i, knn, inv)
    lo = np.minimum(rows, cols)
    hi = np.maximum(rows, cols)
    key = np.unique(lo * n + hi)  # union of both directions, deduplicated
    return np.column_stack((key // n, key % n)).astype(np.int64)


def knn_selected(x, knn: int, sigma: float) -> np.ndarray:
    """Per-row selected neighbour sets (n x knn, unordered within a row)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    inv = -1.0 / (2.0 * sigma**2)
    return np.stack([knn_select_row(x, i, knn, inv) for i in range(x.shape[0])])


def edge_weights(x, e: np.ndarray, sigma: float) -> np.ndarray:
    """exp(-d2 / (2 sigma^2)) once per unordered pair (graph.py:136-141),
    then clamp_zero (graph.py:230-231; a no-op for exp >= 0)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    diff = x[e[:, 0]] - x[e[:, 1]]
    d2 = np.einsum("ij,ij->i", diff, diff)
    return np.maximum(np.exp(-d2 / (2.0 * sigma**2)), 0.0)


def edge_similarity(x, e: np.ndarray, kind: str, negative_policy: str = "clamp_zero") -> np.ndarray:
    """graph.py:136-147 + 229-236 for the cosine / cross_correlation
    measures: one value per (i < j) edge, then the negative policy.  Raises
    ValueError(index) for a degenerate (zero-norm / constant) involved point."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    e = np.asarray(e, dtype=np.int64).reshape(-1, 2)
    xc = x - x.mean(axis=1, keepdims=True) if kind == "cross_correlation" else x
    sq = np.einsum("ij,ij->i", xc, xc)
    bad = np.flatnonzero(sq == 0.0)
    bad = bad[np.isin(bad, np.unique(e))]
    if len(bad):
        raise ValueError(int(bad[0]))
    ei, ej = e[:, 0], e[:, 1]
    v = np.clip(np.einsum("ij,ij->i", xc[ei], xc[ej]) / np.sqrt(sq[ei] * sq[ej]), -1.0, 1.0)
    if negative_policy == "clamp_zero":
        v = np.maximum(v, 0.0)
    elif negative_policy == "abs":
        v = np.abs(v)
    return v


def eps_edges(x, eps: float) -> np.ndarray:
    """graph.py:160-176: pairs (i < j) with d2 <= eps^2, row-major."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    eps2 = eps * eps
    out = []
    for i in range(x.shape[0] - 1):
        d2 = np.einsum("ij,ij->i", x[i + 1:] - x[i], x[i + 1:] - x[i])
        hits = np.flatnonzero(d2 <= eps2) + i + 1
        out.append(np.column_stack((np.full(len(hits), i, dtype=np.int64), hits)))
    return np.concatenate(out) if out else np.empty((0, 2), dtype=np.int64)


def threshold_edges_exp(x, lam: float, sigma: float) -> np.ndarray:
    """graph.py:206-211 with the exp_decay measure (graph.py:149-157):
    pairs (i < j) with exp(inv * d2) > lam."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    inv = -1.0 / (2.0 * sigma**2)
    out = []
    for i in range(x.shape[0] - 1):
        s = np.exp(inv * np.einsum("ij,ij->i", x - x[i], x - x[i]))
        hits = np.flatnonzero(s[i + 1:] > lam) + i + 1
        out.append(np.column_stack((np.full(len(hits), i, dtype=np.int64), hits)))
    return np.concatenate(out) if out else np.empty((0, 2), dtype=np.int64)


def csr_from_edges(n: int, e: np.ndarray, w: np.ndarray):
    """Mirror each pair and sort by (row, col) (graph.py:232-237,
    sparse.py:145-170), then compress rows (sparse.py:182-187)."""
    rows = np.concatenate((e[:, 0], e[:, 1]))
    cols = np.concatenate((e[:, 1], e[:, 0]))
    vals = np.concatenate((w, w))
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    counts = np.bincount(rows, minlength=n)
    row_ptr = np.concatenate(([0], np.cumsum(counts, dtype=np.int64)))
    return row_ptr, cols.astype(np.int64), vals


# --------------------------------------------------------------------------
# sparse / normalisation (sparse.py:195-207, laplacian.py:27-106)
# --------------------------------------------------------------------------
def _row_ids(row_ptr: np.ndarray) -> np.ndarray:
    return np.repeat(np.arange(len(row_ptr) - 1, dtype=np.int64), np.diff(row_ptr))


def spmv_seq(row_ptr, col, vals, x) -> np.ndarray:
    """y = A x with every row summed sequentially in column order
    (sparse.py:205-207: rounded products accumulated by bincount)."""
    n = len(row_ptr) - 1
    return np.bincount(_row_ids(row_ptr), weights=vals * np.asarray(x)[col], minlength=n)


def degrees(row_ptr, col, vals) -> np.ndarray:
    """W 1 (laplacian.py:27-31)."""
    return spmv_seq(row_ptr, col, vals, np.ones(len(row_ptr) - 1))


def sym_scale_vals(row_ptr, col, vals, d) -> np.ndarray:
    """w_ij / sqrt(d_i d_j) (laplacian.py:84-91)."""
    if np.any(d <= 0.0):
        raise ValueError("non-positive degree")
    return vals / np.sqrt(d[_row_ids(row_ptr)] * d[col])


def row_scale_vals(row_ptr, vals, d) -> np.ndarray:
    """laplacian.py:75-81: vals / d[row]."""
    return vals / d[_row_ids(row_ptr)]


def remove_isolated(row_ptr, col, vals, d):
    """laplacian.py:53-64 (policy 'remove'): induced submatrix on d != 0,
    returns (row_ptr, col, vals, d_kept, remap)."""
    n = len(row_ptr) - 1
    keep = d != 0.0
    remap = np.full(n, -1, dtype=np.int64)
    remap[keep] = np.arange(int(keep.sum()), dtype=np.int64)
    rows = _row_ids(row_ptr)
    mask = keep[rows] & keep[col]
    n_new = int(keep.sum())
    counts = np.bincount(remap[rows[mask]], minlength=n_new)
    rp = np.concatenate(([0], np.cumsum(counts, dtype=np.int64)))
    return rp, remap[col[mask]], vals[mask], d[keep], remap


def recover_embedding(u: np.ndarray, d: np.ndarray) -> np.ndarray:
    """v = u / sqrt(d) by rows, unit columns (laplacian.py:94-106)."""
    v = u / np.sqrt(d)[:, None]
    norms = np.linalg.norm(v, axis=0)
    norms[norms == 0.0] = 1.0
    return v / norms


def normalize_rows(v: np.ndarray) -> np.ndarray:
    """pipeline.py:242-245."""
    norms = np.linalg.norm(v, axis=1, keepdims=True)
    norms[norms == 0.0] = 1.0
    return v / norms


# --------------------------------------------------------------------------
# stage 2: thick-restart Lanczos (eigen.py:86-302)
# --------------------------------------------------------------------------
class LanczosFailed(RuntimeError):
    def __init__(self, msg, values=None, residuals=None):
        super().__init__(msg)
        self.values = values
        self.residuals = residuals


def lanczos_topk(apply, n: int, k: int, m: int | None = None, tol: float = 1e-8,
                 max_restarts: int = 300, seed: int = 0):
    """Top-k eigenpairs of a symmetric operator.

    Restates RciSession (eigen.py:94-248) driven as in eigensolve
    (eigen.py:291-302): full CGS2 reorthogonalisation every step
    (eigen.py:131-135, 160-163), breakdown handling (eigen.py:166-176,
    137-150), dense projected eigenproblem and convergence test
    (eigen.py:187-200), verification sweep from a fresh direction
    (eigen.py:181-185, 198-209, 227-229), thick restart with arrowhead
    coupling (eigen.py:218-239) and true residuals (eigen.py:241-248).
    Returns (values, vectors, residuals, stats).
    """
    if m is None:
        m = min(n, max(2 * k, k + 8))  # eigen.py:53-55
    if not (1 <= k < m <= n) or not tol > 0:
        raise ValueError("bad Lanczos configuration")
    rng = np.random.default_rng(seed)
    basis = np.zeros((n, m + 1))
    proj = np.zeros((m, m))
    scale = 0.0
    pending = None
    restarts = 0
    breakdowns = 0
    history = []
    start = rng.standard_normal(n)
    basis[:, 0] = start / np.linalg.norm(start)
    j = 0

    def cgs2(w, count):
        b = basis[:, :count]
        for _ in range(2):
            w = w - b @ (b.T @ w)
        return w

    def fresh(count, is_breakdown=True):
        nonlocal breakdowns
        for _ in range(3):
            v = cgs2(rng.standard_normal(n), count)
            nv = np.linalg.norm(v)
            if nv > 1e-6 * np.sqrt(n):
                if is_breakdown:
                    breakdowns += 1
                return v / nv
        raise LanczosFailed("breakdown: basis cannot be extended")

    while True:
        q = basis[:, j]
        w = np.asarray(apply(q.copy()), dtype=np.float64).copy()
        alpha = q @ w
        proj[j, j] = alpha
        w -= basis[:, :j + 1] @ proj[:j + 1, j]
        w = cgs2(w, j + 1)
        beta = float(np.linalg.norm(w))
        scale = max(scale, abs(alpha), beta)
        if j + 1 < m:
            if beta > BREAKDOWN_RTOL * max(1.0, scale):
                basis[:, j + 1] = w / beta
                proj[j, j + 1] = proj[j + 1, j] = beta
            else:
                basis[:, j + 1] = fresh(j + 1)
                proj[j, j + 1] = proj[j + 1, j] = 0.0
            j += 1
            continue
        theta, s = np.linalg.eigh(proj)
        order = np.argsort(-theta, kind="stable")
        theta, s = theta[order], s[:, order]
        est = beta * np.abs(s[m - 1, :k])
        history.append(float(est.max()))
        converged = bool(np.all(est <= tol * np.maximum(1.0, np.abs(theta[:k]))))
        verified = False
        if pending is not None:
            slack = np.maximum(1.0, np.abs(theta[:k])) * max(tol, 1e-12)
            verified = bool(np.all(np.abs(theta[:k] - pending) <= slack))
        if converged and (m == n or verified):
            vecs = basis[:, :m] @ s[:, :k]
            vecs /= np.linalg.norm(vecs, axis=0)
            vals = theta[:k].copy()
            res = np.array([np.linalg.norm(apply(vecs[:, i]) - vals[i] * vecs[:, i])
                            for i in range(k)])
            stats = dict(restarts=restarts, breakdowns=breakdowns, history=history)
            return vals, vecs, res, stats
        if restarts >= max_restarts:
            raise LanczosFailed("max restarts", values=theta[:k].copy(), residuals=est)
        restarts += 1
        retained = basis[:, :m] @ s[:, :k]
        coupling = beta * s[m - 1, :k]
        basis[:, :k] = retained
        proj[:] = 0.0
        proj[np.arange(k), np.arange(k)] = theta[:k]
        if converged:
            pending = theta[:k].copy()
            basis[:, k] = fresh(k, is_breakdown=False)
        else:
            pending = None
            if beta > BREAKDOWN_RTOL * max(1.0, scale):
                basis[:, k] = w / beta
                proj[:k, k] = coupling
                proj[k, :k] = coupling
            else:
                basis[:, k] = fresh(k)
        j = k


# --------------------------------------------------------------------------
# stage 3: k-means (kmeans.py:84-222)
# --------------------------------------------------------------------------
def pairwise_sq_dist(v: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Gram expansion with einsum cross term, clamped at 0 (kmeans.py:84-98)."""
    vn = np.einsum("ij,ij->i", v, v)
    cn = np.einsum("ij,ij->i", c, c)
    s = vn[:, None] + cn[None, :]
    s -= 2.0 * np.einsum("id,jd->ij", v, c)
    return np.maximum(s, 0.0)


def _dist_to_one(v, c):
    diff = v - c  # kmeans.py:101-104 (direct differences)
    return np.einsum("ij,ij->i", diff, diff)


def kmeanspp_indices(v: np.ndarray, k: int, seed) -> np.ndarray:
    """Row indices chosen by k-means++ seeding (kmeans.py:107-136); the
    reference returns v[chosen], this returns ``chosen`` itself."""
    n = v.shape[0]
    rng = np.random.default_rng(seed)
    chosen = np.empty(k, dtype=np.int64)
    chosen[0] = rng.integers(n)
    taken = np.zeros(n, dtype=bool)
    taken[chosen[0]] = True
    d2 = _dist_to_one(v, v[chosen[0]])
    for i in range(1, k):
        cand = np.flatnonzero(~taken & (d2 > 0.0))
        if len(cand):
            w = d2[cand]
            pick = cand[rng.choice(len(cand), p=w / w.sum())]
        else:
            free = np.flatnonzero(~taken)
            pick = free[rng.integers(len(free))]
        chosen[i] = pick
        taken[pick] = True
        d2 = np.minimum(d2, _dist_to_one(v, v[pick]))
    return chosen


def _update(v, labels, k, cost):
    """kmeans.py:139-156: point-order sums, means, farthest-point reseed."""
    sums = np.zeros((k, v.shape[1]))
    np.add.at(sums, labels, v)
    counts = np.bincount(labels, minlength=k)
    c = np.zeros((k, v.shape[1]))
    ne = counts > 0
    c[ne] = sums[ne] / counts[ne, None]
    empty = np.flatnonzero(counts == 0)
    if len(empty):
        far = np.argsort(-cost, kind="stable")
        for slot, cl in enumerate(empty):
            c[cl] = v[far[slot]]
    return c


def lloyd(v: np.ndarray, init_c: np.ndarray, max_iters: int = 300, tol_changes: int = 0):
    """kmeans.py:159-196. Returns (labels, centroids, sse, iters, sse_history)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    c = np.ascontiguousarray(init_c, dtype=np.float64)
    k, n = c.shape[0], v.shape[0]
    s = pairwise_sq_dist(v, c)
    labels = np.argmin(s, axis=1)
    cost = s[np.arange(n), labels]
    hist = [float(cost.sum())]
    it = 0
    while it < max_iters:
        c = _update(v, labels, k, cost)
        s = pairwise_sq_dist(v, c)
        new = np.argmin(s, axis=1)
        cost = s[np.arange(n), new]
        hist.append(float(cost.sum()))
        it += 1
        changes = int(np.count_nonzero(new != labels))
        labels = new
        if changes <= tol_changes:
            break
    return labels, c, hist[-1], it, np.array(hist)


def kmeans(v: np.ndarray, k: int, seed: int = 0, max_iters: int = 300,
           tol_changes: int = 0, restarts: int = 1, init: str = "kmeanspp"):
    """kmeans.py:199-222 (best of ``restarts`` by SSE, derived seeds)."""
    v = np.ascontiguousarray(v, dtype=np.float64)

    def once(sd):
        if init == "kmeanspp":
            ic = v[kmeanspp_indices(v, k, sd)]
        else:
            ic = v[np.random.default_rng(sd).choice(v.shape[0], size=k, replace=False)]
        return lloyd(v, ic, max_iters, tol_changes)

    best = once(seed)
    for r in range(1, restarts):
        sd = int(np.random.SeedSequence([seed, r]).generate_state(1)[0])
        cand = once(sd)
        if cand[2] < best[2]:
            best = cand
    return best


# --------------------------------------------------------------------------
# metrics (metrics.py:34-99)
# --------------------------------------------------------------------------
def ncut(row_ptr, col, vals, labels) -> float:
    lab = np.asarray(labels, dtype=np.int64)
    n = len(row_ptr) - 1
    k = int(lab.max()) + 1
    rows = _row_ids(row_ptr)
    deg = np.bincount(rows, weights=vals, minlength=n)
    vol = np.bincount(lab, weights=deg, minlength=k)
    crossing = lab[rows] != lab[col]
    bnd = np.bincount(lab[rows[crossing]], weights=vals[crossing], minlength=k)
    if np.any(vol <= 0.0):
        raise ValueError("zero-volume part")
    return 0.5 * float((bnd / vol).sum())


def cut(row_ptr, col, vals, labels) -> float:
    """metrics.py:42-48: half the weight of the crossing entries."""
    lab = np.asarray(labels, dtype=np.int64)
    crossing = lab[_row_ids(row_ptr)] != lab[col]
    return 0.5 * float(vals[crossing].sum())


def ratio_cut(row_ptr, col, vals, labels, k: int) -> float:
    """metrics.py:51-56: half the sum of boundary weight / part size
    (ValueError for an empty part, EmptyPart in the package)."""
    lab = np.asarray(labels, dtype=np.int64)
    sizes = np.bincount(lab, minlength=k)
    if np.any(sizes == 0):
        raise ValueError("empty part")
    rows = _row_ids(row_ptr)
    crossing = lab[rows] != lab[col]
    bnd = np.bincount(lab[rows[crossing]], weights=vals[crossing], minlength=k)
    return 0.5 * float((bnd / sizes).sum())


def ari(a, b) -> float:
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    n = len(a)
    if n == 0:
        return 1.0
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    kb = int(bi.max()) + 1
    cont = np.bincount(ai * kb + bi, minlength=(int(ai.max()) + 1) * kb)
    comb = lambda t: (t.astype(np.float64) * (t - 1.0) / 2.0).sum()  # noqa: E731
    cont = cont.reshape(-1, kb)
    sc, sr, sk = comb(cont), comb(cont.sum(axis=1)), comb(cont.sum(axis=0))
    total = n * (n - 1.0) / 2.0
    exp = sr * sk / total if total > 0 else 0.0
    mx = 0.5 * (sr + sk)
    if mx == exp:
        return 1.0
    return float((sc - exp) / (mx - exp))


# --------------------------------------------------------------------------
# end to end (pipeline.py:211-267, PointsInput knn + exp_decay)
# --------------------------------------------------------------------------
def run_points(x, knn: int, sigma: float, k: int, normalize: bool = True,
               eigen_seed: int = 0, kmeans_seed: int = 0, tol: float = 1e-8, timings=None):
    import time

    t = time.perf_counter
    t0 = t()
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    e = knn_edges(x, knn, sigma)
    row_ptr, col, vals = csr_from_edges(n, e, edge_weights(x, e, sigma))
    t1 = t()
    d = degrees(row_ptr, col, vals)
    if np.any(d == 0.0):
        raise ValueError("isolated node")
    t2 = t()
    a = sym_scale_vals(row_ptr, col, vals, d)
    apply = lambda z: spmv_seq(row_ptr, col, a, z)  # noqa: E731
    values, vectors, residuals, stats = lanczos_topk(apply, n, k, tol=tol, seed=eigen_seed)
    emb = recover_embedding(vectors, d)
    t3 = t()
    rows = normalize_rows(emb) if normalize else emb
    chosen = kmeanspp_indices(rows, k, kmeans_seed)
    labels, cent, sse, iters, hist = lloyd(rows, rows[chosen])
    t4 = t()
    _, compact = np.unique(labels, return_inverse=True)
    nc = ncut(row_ptr, col, vals, compact)
    t5 = t()
    if timings is not None:
        timings.update(graph=t1 - t0, degrees=t2 - t1, eigen=t3 - t2, kmeans=t4 - t3,
                       metrics=t5 - t4)
    return dict(row_ptr=row_ptr, col=col, vals=vals, degrees=d, values=values,
                vectors=vectors, residuals=residuals, embedding=rows, chosen=chosen,
                labels=labels, centroids=cent, sse=sse, iters=iters, sse_history=hist,
                ncut=nc, eigen_stats=stats)
