"""k-means++ seeding and Lloyd iterations (drop-in for speclust.kmeans).

All O(n k d) and O(n d) work runs on the GPU:
  * assignment: fp64 Gram-expansion distance tiles with a fused argmin
    (ties -> lowest centroid index) and clamp at zero (kmeans.py:84-98);
  * update: stable bucketing by label, then per (cluster, feature) sums in
    point order — the order of the reference's ``np.add.at`` — divided by
    the counts; empty clusters take the farthest points (kmeans.py:139-156);
  * k-means++: device distance update / candidate reduction / cumulative
    draw; the host keeps the numpy PCG64 stream so the draws are the
    reference's own (kmeans.py:107-136).
"""

from __future__ import annotations

from dataclasses import dataclass

import os
import sys
import time

import numpy as np

from . import _native as nat
from .errors import BadConfig, DimensionMismatch

__all__ = ["KmeansConfig", "Labeling", "pairwise_sq_dist", "kmeanspp_init", "lloyd", "kmeans"]

INIT_KINDS = ("kmeanspp", "random_points")


@dataclass(frozen=True)
class KmeansConfig:
    k: int
    max_iters: int = 300
    seed: int = 0
    init: str = "kmeanspp"
    tol_changes: int = 0
    restarts: int = 1

    def __post_init__(self):
        checks = (
            (self.k >= 1, f"k must be >= 1, got {self.k}"),
            (self.max_iters >= 1, f"max_iters must be >= 1, got {self.max_iters}"),
            (self.tol_changes >= 0, f"tol_changes must be >= 0, got {self.tol_changes}"),
            (self.init in INIT_KINDS, f"unknown init {self.init!r}"),
            (self.restarts >= 1, f"restarts must be >= 1, got {self.restarts}"),
        )
        for ok, msg in checks:
            if not ok:
                raise BadConfig(msg)


@dataclass(frozen=True)
class Labeling:
    labels: np.ndarray
    centroids: np.ndarray
    sse: float
    iters_run: int
    sse_history: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "labels", nat.frozen(np.asarray(self.labels, dtype=np.int64)))
        for name in ("centroids", "sse_history"):
            object.__setattr__(self, name, nat.frozen(np.asarray(getattr(self, name), dtype=np.float64)))


def _as_2d(a, what: str):
    torch = nat.torch_cuda()
    if isinstance(a, torch.Tensor):
        if a.ndim != 2:
            raise DimensionMismatch(f"{what} must be 2-D, got ndim={a.ndim}")
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    h = np.ascontiguousarray(a, dtype=np.float64)
    if h.ndim != 2:
        raise DimensionMismatch(f"{what} must be 2-D, got ndim={h.ndim}")
    return nat.to_device(h, torch.float64)


def _same_d(v, c):
    if v.shape[1] != c.shape[1]:
        raise DimensionMismatch(f"dimension mismatch: points have d={v.shape[1]}, centroids d={c.shape[1]}")


def pairwise_sq_dist(v, c) -> np.ndarray:
    """n x k squared distances by Gram expansion, clamped at 0."""
    torch = nat.torch_cuda()
    vd, cd = _as_2d(v, "points"), _as_2d(c, "centroids")
    _same_d(vd, cd)
    n, d = vd.shape
    k = cd.shape[0]
    out = torch.empty((n, k), dtype=torch.float64, device="cuda")
    nat.check(nat.load().sc_pairwise_sq_dist(n, k, d, nat.ptr(vd), nat.ptr(cd), nat.ptr(out), nat.stream_handle()))
    return nat.to_host(out)


def kmeanspp_indices_device(vd, k: int, seed) -> np.ndarray:
    """Row indices of the k-means++ seeding (kmeans.py:107-136) for the
    CUDA (n, d) tensor ``vd``; the random draws come from numpy's
    default_rng(seed), consumed exactly as the reference consumes them."""
    n, d = vd.shape
    if not 1 <= k <= n:
        raise BadConfig(f"k must satisfy 1 <= k <= n, got k={k}, n={n}")
    lib = nat.load()
    rng = np.random.default_rng(seed)
    h = nat.vp()
    nat.check(lib.sc_kmeanspp_create(n, d, nat.ptr(vd), nat.stream_handle(), nat.C.byref(h)))
    try:
        chosen = np.empty(k, dtype=np.int64)
        chosen[0] = rng.integers(n)
        nat.check(lib.sc_kmeanspp_take(h, int(chosen[0])))
        cnt, nfree, pick = nat.C.c_int64(0), nat.C.c_int64(0), nat.C.c_int64(0)
        for i in range(1, k):
            nat.check(lib.sc_kmeanspp_candidates(h, nat.C.byref(cnt), nat.C.byref(nfree)))
            if cnt.value > 0:
                u = rng.random()  # Generator.choice(len, p=...) draws one double
                nat.check(lib.sc_kmeanspp_pick(h, 0, u, 0, nat.C.byref(pick)))
            else:
                r = int(rng.integers(nfree.value))
                nat.check(lib.sc_kmeanspp_pick(h, 1, 0.0, r, nat.C.byref(pick)))
            chosen[i] = pick.value
        return chosen
    finally:
        lib.sc_kmeanspp_destroy(h)


def kmeanspp_init(v, k: int, seed) -> np.ndarray:
    """k distinct rows of v by D^2 sampling (kmeans.py:107-136)."""
    vd = _as_2d(v, "points")
    idx = kmeanspp_indices_device(vd, k, seed)
    return nat.to_host(vd[nat.to_device(idx, nat.torch_cuda().int64)])


def lloyd_device(vd, cd, cfg: KmeansConfig):
    """Lloyd iterations on device tensors; returns (labels tensor, centroids
    tensor, sse_history numpy, iters)."""
    torch = nat.torch_cuda()
    _same_d(vd, cd)
    n, d = vd.shape
    k = cd.shape[0]
    labels = torch.empty(n, dtype=torch.int64, device="cuda")
    cent = torch.empty((k, d), dtype=torch.float64, device="cuda")
    hist = np.zeros(cfg.max_iters + 1)
    iters = nat.C.c_int64(0)
    nat.check(nat.load().sc_lloyd(n, d, k, nat.ptr(vd), nat.ptr(cd), cfg.max_iters, cfg.tol_changes,
                                  nat.ptr(labels), nat.ptr(cent), hist.ctypes.data_as(nat.P_f64),
                                  nat.C.byref(iters), nat.stream_handle()))
    it = int(iters.value)
    return labels, cent, hist[: it + 1].copy(), it


def lloyd(v, init_c, cfg: KmeansConfig) -> Labeling:
    """Lloyd iterations from the given centroids (kmeans.py:159-196)."""
    vd, cd = _as_2d(v, "points"), _as_2d(init_c, "centroids")
    labels, cent, hist, it = lloyd_device(vd, cd, cfg)
    return Labeling(nat.to_host(labels), nat.to_host(cent), float(hist[-1]), it, hist)


def _init_rows(vd, cfg: KmeansConfig, seed) -> np.ndarray:
    if cfg.init == "kmeanspp":
        return kmeanspp_indices_device(vd, cfg.k, seed)
    rng = np.random.default_rng(seed)
    return rng.choice(vd.shape[0], size=cfg.k, replace=False)


def kmeans_device(vd, cfg: KmeansConfig):
    """Best of ``cfg.restarts`` runs by SSE (kmeans.py:199-222) on a CUDA
    tensor; returns (labels, centroids, sse_history, iters)."""
    torch = nat.torch_cuda()
    if cfg.k > vd.shape[0]:
        raise BadConfig(f"k={cfg.k} exceeds number of points n={vd.shape[0]}")
    best = None
    dbg = os.environ.get("SPECLUST_TIMING_DEBUG") is not None
    for r in range(cfg.restarts):
        seed = cfg.seed if r == 0 else int(np.random.SeedSequence([cfg.seed, r]).generate_state(1)[0])
        t0 = time.perf_counter()
        rows = _init_rows(vd, cfg, seed)
        init_c = vd[torch.from_numpy(np.asarray(rows, dtype=np.int64)).to("cuda")].contiguous()
        if dbg:
            torch.cuda.synchronize()
            t1 = time.perf_counter()
        cand = lloyd_device(vd, init_c, cfg)
        if dbg:
            torch.cuda.synchronize()
            print(f"[kmeans] init {t1 - t0:.3f} s, lloyd {time.perf_counter() - t1:.3f} s ({cand[3]} iterations)",
                  file=sys.stderr)
        if best is None or cand[2][-1] < best[2][-1]:
            best = cand
    return best


def kmeans(v, cfg: KmeansConfig) -> Labeling:
    """k-means++ (or distinct random rows) + Lloyd, best of restarts."""
    vd = _as_2d(v, "points")
    labels, cent, hist, it = kmeans_device(vd, cfg)
    return Labeling(nat.to_host(labels), nat.to_host(cent), float(hist[-1]), it, hist)
