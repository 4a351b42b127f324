"""Similarity-graph construction (drop-in for speclust.graph).

The north-star pattern — union kNN with the Gaussian ``exp_decay`` measure —
runs entirely on the GPU (``sc_knn_graph_f64``): low-precision distance
tiles with a streaming per-row top-R list, an exact fp64 recheck certified by
an error bound, an exact fallback for uncertified rows, and union
symmetrisation written straight into CSR.  The ranking key and edge values
follow graph.py:149-157 / 136-141 of the reference.

The other measures (cosine, cross-correlation) over a given edge list and the
eps / threshold patterns run on the GPU as well
(sc_patterns.cu); the kNN pattern with cosine / cross-correlation runs the
same tensor-core candidate scan on row-normalised operands with a
cosine-space certificate (``sc_knn_graph_measure_f64``).  There is no host
fallback anywhere.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import DegenerateVector, DimensionMismatch, InvalidFormat
from .sparse import CooMatrix, DeviceCsr, coo_canonicalize

__all__ = [
    "SimilarityMeasure",
    "similarity",
    "build_edges_eps",
    "build_edges_knn",
    "build_edges_threshold",
    "build_similarity",
    "validate_edges",
    "knn_graph_device",
]

MEASURE_KINDS = ("cosine", "cross_correlation", "exp_decay")
NEGATIVE_POLICIES = ("clamp_zero", "abs", "keep")


@dataclass(frozen=True)
class SimilarityMeasure:
    """Measure selector; ``sigma`` is the Gaussian width of exp_decay
    (reference graph.py:32-57)."""

    kind: str
    sigma: float | None = None

    def __post_init__(self):
        if self.kind not in MEASURE_KINDS:
            raise ValueError(f"unknown measure kind {self.kind!r}")
        if self.kind == "exp_decay" and (self.sigma is None or not self.sigma > 0):
            raise ValueError("exp_decay requires sigma > 0")

    @classmethod
    def cosine(cls) -> "SimilarityMeasure":
        return cls("cosine")

    @classmethod
    def cross_correlation(cls) -> "SimilarityMeasure":
        return cls("cross_correlation")

    @classmethod
    def exp_decay(cls, sigma: float) -> "SimilarityMeasure":
        return cls("exp_decay", sigma)

    def two_sigma_sq(self) -> float:
        # evaluated exactly as the reference writes it: 2.0 * sigma**2
        return 2.0 * self.sigma**2


def as_points(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise InvalidFormat("point matrix must be 2-D with n >= 1, d >= 1")
    if not np.isfinite(a).all():
        raise InvalidFormat("point matrix must be finite")
    return a


def validate_edges(pairs, n: int) -> np.ndarray:
    """(m, 2) int64 edge list without self-loops, out-of-range indices or
    repeated unordered pairs (reference graph.py:70-84)."""
    e = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if len(e):
        if e.min() < 0 or e.max() >= n:
            raise InvalidFormat("edge index out of range")
        if (e[:, 0] == e[:, 1]).any():
            raise InvalidFormat("edge list contains a self-loop")
        key = np.minimum(e[:, 0], e[:, 1]) * n + np.maximum(e[:, 0], e[:, 1])
        if len(np.unique(key)) != len(key):
            raise InvalidFormat("edge list contains a duplicate unordered pair")
    return e


def similarity(x_i, x_j, m: SimilarityMeasure) -> float:
    """Scalar similarity of two vectors (reference graph.py:107-133); a
    convenience helper, not part of the device path."""
    a = np.asarray(x_i, dtype=np.float64)
    b = np.asarray(x_j, dtype=np.float64)
    if a.ndim != 1 or a.shape != b.shape:
        raise DimensionMismatch(f"vectors must be 1-D of equal length, got {a.shape} and {b.shape}")
    if a.shape[0] < 1:
        raise DimensionMismatch("vectors must have d >= 1")
    if m.kind == "exp_decay":
        return float(np.exp(-float(np.sum((a - b) ** 2)) / m.two_sigma_sq()))
    if m.kind == "cross_correlation":
        a, b = a - a.mean(), b - b.mean()
    sa, sb = float(a @ a), float(b @ b)
    for s, side in ((sa, "left"), (sb, "right")):
        if s == 0.0:
            raise DegenerateVector(f"{side} vector is degenerate for {m.kind}", index=None)
    return float(np.clip((a @ b) / np.sqrt(sa * sb), -1.0, 1.0))


def _require_exp_decay(m: SimilarityMeasure, what: str):
    if m.kind != "exp_decay":
        raise NotImplementedError(
            f"{what} with measure {m.kind!r}: the sharded kNN stages support exp_decay only "
            "(single-GPU knn_graph_device handles every measure)"
        )


def _knn_graph_corr(xd, knn: int, m: SimilarityMeasure, negative_policy: str, return_stats: bool):
    """kNN graph with the cosine / cross-correlation measure
    (sc_knn_graph_measure_f64): ranking by the reference's similarity,
    values under the negative policy."""
    torch = nat.torch_cuda()
    n, d = xd.shape
    cap = 2 * n * knn
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(cap, dtype=torch.int32, device="cuda")
    vals = torch.empty(cap, dtype=torch.float64, device="cuda")
    nnz, deg = nat.C.c_int64(), nat.C.c_int64()
    stats = (nat.C.c_int64 * 8)()
    rc = nat.load().sc_knn_graph_measure_f64(n, d, nat.ptr(xd), knn, 1 if m.kind == "cosine" else 2, 1.0,
                                             NEGATIVE_POLICIES.index(negative_policy), nat.ptr(rp), nat.ptr(col),
                                             nat.ptr(vals), nat.C.byref(nnz), stats, nat.C.byref(deg),
                                             nat.stream_handle())
    if rc != 0 and deg.value >= 0:
        what = "constant" if m.kind == "cross_correlation" else "zero"
        raise DegenerateVector(f"{what} vector at point index {deg.value} is invalid for {m.kind}",
                               index=int(deg.value))
    nat.check(rc)
    w = DeviceCsr(n, n, rp, col[: nnz.value].clone(), vals[: nnz.value].clone())
    if return_stats:
        keys = ("list_R", "list_cap", "fallback_rows")
        out = {key: int(stats[i]) for i, key in enumerate(keys)}
        out["nnz"] = w.nnz
        return w, out
    return w


def knn_graph_device(x, knn: int, m: SimilarityMeasure, return_stats: bool = False,
                     negative_policy: str = "clamp_zero"):
    """Union-kNN similarity matrix W as a DeviceCsr, built on the GPU in one
    call (graph.py:185-237 + sparse.py:182-187 fused).  exp_decay keeps the
    kNN locality scan order on W (``locality_perm``) for the eigensolver;
    cosine / cross_correlation go through sc_knn_graph_measure_f64.

    ``x`` may be a numpy array or a CUDA float64 tensor (n x d)."""
    if negative_policy not in NEGATIVE_POLICIES:
        raise ValueError(f"unknown negative_policy {negative_policy!r}")
    torch = nat.torch_cuda()
    if isinstance(x, torch.Tensor):
        # CUDA tensors are used in place; host tensors (e.g. pinned) are copied
        xd = x.to(device="cuda", dtype=torch.float64, non_blocking=True).contiguous()
        n, d = xd.shape
    else:
        xh = as_points(x)
        n, d = xh.shape
        xd = nat.to_device(xh, torch.float64)
    if not 1 <= knn < n:
        raise ValueError(f"knn must satisfy 1 <= knn < n, got {knn} for n={n}")
    if m.kind != "exp_decay":
        return _knn_graph_corr(xd, knn, m, negative_policy, return_stats)
    # selection (sc_knn_select_f64) + union (sc_knn_union_f64) == sc_knn_graph_f64;
    # the two-stage form keeps the locality scan order for the eigensolver
    # the selection also returns each slot's exact d2, so the union fills the
    # CSR values without recomputing distances
    sel = torch.empty((n, knn), dtype=torch.int32, device="cuda")
    sel_vals = torch.empty((n, knn), dtype=torch.float64, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    stats = (nat.C.c_int64 * 8)()
    lib = nat.load()
    nat.check(lib.sc_knn_select_vals_f64(n, d, nat.ptr(xd), knn, m.two_sigma_sq(), 0, n, nat.ptr(sel),
                                         nat.ptr(sel_vals), nat.ptr(perm), stats, nat.stream_handle()))
    w = knn_union_device(xd, knn, m, sel, perm, 0, n, sel_vals)
    del sel, sel_vals
    w.locality_perm = perm  # scan position -> point
    if return_stats:
        keys = ("list_R", "list_cap", "fallback_rows")
        out = {key: int(stats[i]) for i, key in enumerate(keys)}
        out["nnz"] = w.nnz
        return w, out
    return w


def _points_device(x):
    torch = nat.torch_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float64, non_blocking=True).contiguous()
    return nat.to_device(as_points(x), torch.float64)


def knn_select_device(x, knn: int, m: SimilarityMeasure, p0: int, p1: int, with_vals: bool = False):
    """Selection stage of the kNN graph for the points at scan positions
    [p0, p1) (sc_knn_select_f64): returns (sel (p1-p0, knn) int32 CUDA,
    perm (n,) int32 CUDA scan order), plus with ``with_vals`` each slot's
    exact d2 (p1-p0, knn) fp64 (sc_knn_select_vals_f64) for the
    value-carrying union."""
    _require_exp_decay(m, "knn graph")
    torch = nat.torch_cuda()
    xd = _points_device(x)
    n, d = xd.shape
    if not 1 <= knn < n:
        raise ValueError(f"knn must satisfy 1 <= knn < n, got {knn} for n={n}")
    sel = torch.empty((max(p1 - p0, 1), knn), dtype=torch.int32, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    if with_vals:
        vals = torch.empty((max(p1 - p0, 1), knn), dtype=torch.float64, device="cuda")
        nat.check(nat.load().sc_knn_select_vals_f64(n, d, nat.ptr(xd), knn, m.two_sigma_sq(), p0, p1, nat.ptr(sel),
                                                    nat.ptr(vals), nat.ptr(perm), None, nat.stream_handle()))
        return sel[: p1 - p0], perm, vals[: p1 - p0]
    nat.check(nat.load().sc_knn_select_f64(n, d, nat.ptr(xd), knn, m.two_sigma_sq(), p0, p1, nat.ptr(sel),
                                           nat.ptr(perm), None, nat.stream_handle()))
    return sel[: p1 - p0], perm


def knn_union_device(x, knn: int, m: SimilarityMeasure, sel, perm, r0: int, r1: int,
                     sel_vals=None) -> DeviceCsr:
    """Union stage: CSR rows [r0, r1) of W (global columns) from the full
    scan-order selection (sc_knn_union_f64; with ``sel_vals``, the exact
    per-slot d2 of the selection, sc_knn_union_vals_f64 fills the values
    without recomputing distances)."""
    torch = nat.torch_cuda()
    xd = _points_device(x)
    n, d = xd.shape
    nl = r1 - r0
    row_ptr = torch.empty(nl + 1, dtype=torch.int64, device="cuda")
    nnz = nat.C.c_int64(0)
    lib = nat.load()
    cap = 2 * nl * knn + 1024
    for _ in range(2):  # a shard whose reverse edges exceed 2*knn per row retries at the exact size
        col = torch.empty(cap, dtype=torch.int32, device="cuda")
        vals = torch.empty(cap, dtype=torch.float64, device="cuda")
        rc = lib.sc_knn_union_vals_f64(n, d, nat.ptr(xd), knn, m.two_sigma_sq(), nat.ptr(sel),
                                       None if sel_vals is None else nat.ptr(sel_vals), nat.ptr(perm), r0, r1,
                                       nat.ptr(row_ptr), nat.ptr(col), nat.ptr(vals), cap, nat.C.byref(nnz),
                                       nat.stream_handle())
        if rc == 0:
            k = nnz.value
            return DeviceCsr(nl, n, row_ptr, col[:k], vals[:k])
        if nnz.value <= cap:
            nat.check(rc)
        cap = nnz.value
    nat.check(rc)


def build_edges_knn(x, knn: int, m: SimilarityMeasure) -> np.ndarray:
    """Union kNN pattern as (i, j) pairs with i < j in row-major order
    (reference graph.py:185-204), computed on the GPU."""
    x = as_points(x)
    n = x.shape[0]
    if not 1 <= knn < n:
        raise ValueError(f"knn must satisfy 1 <= knn < n, got {knn} for n={n}")
    w = knn_graph_device(x, knn, m, negative_policy="keep")
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(nat.to_host(w.row_ptr)))
    cols = nat.to_host(w.col, np.int64)
    upper = cols > rows
    return np.column_stack((rows[upper], cols[upper]))


def _pattern_edges(x: np.ndarray, mode: int, a: float, b: float) -> np.ndarray:
    """(i < j) pairs of the eps / threshold patterns, computed on the GPU
    (sc_pattern_edges_f64: count, then fill)."""
    torch = nat.torch_cuda()
    n, d = x.shape
    xd = nat.to_device(x, torch.float64)
    lib = nat.load()
    m, deg = nat.C.c_int64(), nat.C.c_int64()
    rc = lib.sc_pattern_edges_f64(n, d, nat.ptr(xd), mode, a, b, None, nat.C.byref(m), nat.C.byref(deg),
                                  nat.stream_handle())
    if rc != 0 and deg.value >= 0:
        raise DegenerateVector(nat.last_error(), index=int(deg.value))
    nat.check(rc)
    if m.value == 0:
        return np.empty((0, 2), dtype=np.int64)
    out = torch.empty((m.value, 2), dtype=torch.int64, device="cuda")
    nat.check(lib.sc_pattern_edges_f64(n, d, nat.ptr(xd), mode, a, b, nat.ptr(out), nat.C.byref(m),
                                       nat.C.byref(deg), nat.stream_handle()))
    return nat.to_host(out)


def build_edges_eps(x, eps: float) -> np.ndarray:
    """Pairs (i, j), i < j, with Euclidean distance at most ``eps``
    (reference graph.py:160-176); d2 in numpy's einsum order on the GPU."""
    x = as_points(x)
    if not eps > 0:
        raise ValueError("eps must be positive")
    return _pattern_edges(x, 0, float(eps), 0.0)


def build_edges_threshold(x, lam: float, m: SimilarityMeasure) -> np.ndarray:
    """Pairs (i, j), i < j, whose similarity strictly exceeds ``lam``
    (reference graph.py:206-211), on the GPU.  exp_decay: the reference's
    exp(inv * d2) with d2 in the einsum order; cosine / cross_correlation:
    dot / sqrt(sq_i sq_j) with the dot in the einsum order (the reference
    forms these with a BLAS GEMM, so pairs within rounding of lam may differ)."""
    x = as_points(x)
    if m.kind == "exp_decay":
        return _pattern_edges(x, 1, float(lam), float(m.sigma))
    return _pattern_edges(x, 2 if m.kind == "cosine" else 3, float(lam), 0.0)


def build_similarity(x, e, m: SimilarityMeasure, negative_policy: str = "clamp_zero") -> CooMatrix:
    """Symmetric similarity matrix over a given edge pattern: one value per
    unordered pair, mirrored (reference graph.py:214-237).  Values are
    computed on the GPU for every measure."""
    x = as_points(x)
    n = x.shape[0]
    e = validate_edges(e, n)
    if negative_policy not in NEGATIVE_POLICIES:
        raise ValueError(f"unknown negative_policy {negative_policy!r}")
    vals = _pair_weights(x, e, m, negative_policy)
    rows = np.concatenate((e[:, 0], e[:, 1]))
    cols = np.concatenate((e[:, 1], e[:, 0]))
    return coo_canonicalize(CooMatrix(n, n, rows, cols, np.concatenate((vals, vals))), dup_policy="error")


def _pair_weights(x: np.ndarray, e: np.ndarray, m: SimilarityMeasure,
                  negative_policy: str = "clamp_zero") -> np.ndarray:
    torch = nat.torch_cuda()
    if len(e) == 0:
        return np.zeros(0)
    xd = nat.to_device(x, torch.float64)
    ed = nat.to_device(e.astype(np.int64), torch.int64)
    out = torch.empty(len(e), dtype=torch.float64, device="cuda")
    lib = nat.load()
    if m.kind == "exp_decay":
        # exp >= 0: clamp_zero / abs / keep are all identities (graph.py:230-233)
        nat.check(lib.sc_pair_weights(x.shape[0], x.shape[1], nat.ptr(xd), len(e), nat.ptr(ed), m.two_sigma_sq(),
                                      nat.ptr(out), nat.stream_handle()))
        return nat.to_host(out)
    deg = nat.C.c_int64()
    rc = lib.sc_edge_similarity_f64(x.shape[0], x.shape[1], nat.ptr(xd), len(e), nat.ptr(ed),
                                    1 if m.kind == "cosine" else 2, NEGATIVE_POLICIES.index(negative_policy),
                                    nat.ptr(out), nat.C.byref(deg), nat.stream_handle())
    if rc != 0 and deg.value >= 0:
        what = "constant" if m.kind == "cross_correlation" else "zero"
        raise DegenerateVector(f"{what} vector at point index {deg.value} is invalid for {m.kind}",
                               index=int(deg.value))
    nat.check(rc)
    return nat.to_host(out)
