"""Sharded spectral clustering across the GPUs of one node.

One process per GPU; ``torch.distributed`` (NCCL over NVLink) carries the
collectives.  The path shards the way SURVEY.md §8(e) prescribes:

* eigen: row-block CSR of A = D^-1/2 W D^-1/2 and row-block Krylov basis.
  Per SpMV one all-gather of the current Lanczos vector; per classical
  Gram-Schmidt pass one all-reduce of the local B^T w (and of |w|^2).  The
  projected matrix T, the convergence / verification / restart decisions and
  the projected eigensolve are replicated: every rank sees bit-identical
  reduced values, so every rank takes the same branch (eigen.py:152-239).
  Start and fresh vectors are drawn per global element (Philox), so the
  sharded solver starts from the same vectors as the single-GPU one.
* k-means: point shards.  Per Lloyd iteration one all-reduce of the
  per-cluster sums and counts, of the change count and of the SSE
  (kmeans.py:159-196); empty clusters take the globally farthest points.
  k-means++ keeps the reference's numpy stream on every rank (identical
  draws, no RNG traffic); the D^2 sample is located by an all-gather of the
  per-shard weight sums (kmeans.py:119-132).
* graph: query tiles (in the locality scan order) are split over ranks; each
  rank scans its tiles against all points (X is replicated), one all-gather
  of the n x knn int32 selection carries the reverse edges, and each rank
  writes its own CSR row block (graph.py:185-237).

The drivers are written against two small interfaces — ``Comm`` (the
collectives) and an *ops* object (per-shard compute).  ``CudaOps`` calls the
C ABI of libspeclust_b200 and is the product path; tests/ supply a numpy ops
object so the distributed logic runs on CPU under gloo.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .eigen import LanczosConfig, default_subspace_dim
from .errors import (BadConfig, Breakdown, EigenNotConverged, IsolatedNode, MaxRestartsExceeded, NotSymmetric,
                     ZeroVolumePart)
from .kmeans import KmeansConfig, Labeling
from .sparse import DeviceCsr

__all__ = ["Comm", "row_bounds", "CudaOps", "lanczos_sharded", "kmeanspp_sharded", "lloyd_sharded", "run_sharded"]

BREAKDOWN_RTOL = 1e-13  # eigen.py:50
REORTH_ETA = 0.05  # second CGS pass threshold (sc_lanczos.cu kReorthEta)

# diagnostics of the last run_sharded call (global nnz, eigen statistics)
last_info: dict = {}


def row_bounds(n: int, world: int) -> list[int]:
    """Contiguous, balanced row blocks: rank r owns [b[r], b[r+1])."""
    return [(r * n) // world for r in range(world + 1)]


class Comm:
    """Collectives over a torch.distributed group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, device, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group, self.device = torch, dist, group, device
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:  # single process
            self.rank, self.world = 0, 1

    def sum_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def gather_rows(self, local, bounds):
        """All-gather of row blocks of different sizes along dim 0."""
        if self.world == 1:
            return local
        torch = self.torch
        sizes = [bounds[r + 1] - bounds[r] for r in range(self.world)]
        mx = max(sizes)
        pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([parts[r][: sizes[r]] for r in range(self.world)], dim=0)

    def gather_scalars(self, values) -> np.ndarray:
        """All-gather of a small float64 vector per rank -> (world, len) host array."""
        torch = self.torch
        t = torch.tensor(np.asarray(values, dtype=np.float64), device=self.device)
        if self.world == 1:
            return t.cpu().numpy()[None, :]
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts).cpu().numpy()

    def exchange_rows(self, local, dest_rank, dest_idx, out_rows: int):
        """Row permutation across ranks: row i of ``local`` goes to rank
        dest_rank[i] as its row dest_idx[i]; returns this rank's (out_rows,
        ...) result.  One all-to-all (counts first); gloo has no CUDA
        all-to-all, so there the payload is staged through host memory."""
        torch = self.torch
        out = torch.empty((out_rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        if self.world == 1:
            out[dest_idx.long()] = local
            return out
        order = torch.argsort(dest_rank, stable=True)
        send, send_idx = local[order].contiguous(), dest_idx[order].to(torch.int64).contiguous()
        in_splits = torch.bincount(dest_rank.long(), minlength=self.world)
        counts = torch.empty(self.world * self.world, dtype=torch.int64, device=in_splits.device)
        self.dist.all_gather_into_tensor(counts, in_splits.to(torch.int64), group=self.group) if \
            local.device.type == "cuda" and self.dist.get_backend(self.group) == "nccl" else \
            self._all_gather_flat(counts, in_splits.to(torch.int64))
        cm = counts.view(self.world, self.world).cpu()
        ins = cm[self.rank].tolist()
        outs = cm[:, self.rank].tolist()
        host = local.device.type == "cuda" and self.dist.get_backend(self.group) != "nccl"
        dev = torch.device("cpu") if host else local.device
        recv = torch.empty((sum(outs),) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
        recv_idx = torch.empty(sum(outs), dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(recv, send.to(dev), outs, ins, group=self.group)
        self.dist.all_to_all_single(recv_idx, send_idx.to(dev), outs, ins, group=self.group)
        out[recv_idx.to(out.device)] = recv.to(out.device)
        return out

    def _all_gather_flat(self, out, t):
        parts = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        out.copy_(self.torch.cat(parts))

    def bcast_(self, t, src):
        if self.world > 1:
            self.dist.broadcast(t, src=src, group=self.group)
        return t


# ---------------------------------------------------------------------------
# per-shard compute through the C ABI (the product path)
class CudaOps:
    """Per-shard operations on CUDA tensors via libspeclust_b200."""

    def __init__(self):
        self.torch = nat.torch_cuda()
        self.lib = nat.load()
        self.device = "cuda"

    def _s(self):
        return nat.stream_handle()

    def zeros(self, shape, dtype=None):
        return self.torch.zeros(shape, dtype=dtype or self.torch.float64, device="cuda")

    def ones(self, n):
        return self.torch.ones(n, dtype=self.torch.float64, device="cuda")

    def to_dev(self, a, dtype=None):
        return nat.to_device(a, dtype or self.torch.float64)

    def host(self, t):
        return nat.to_host(t)

    # ---- graph / normalisation
    def knn_graph(self, x, knn, measure):
        from .graph import knn_graph_device

        return knn_graph_device(x, knn, measure)

    def points(self, x):
        from .graph import _points_device

        return _points_device(x)

    carries_vals = True  # the selection hands each slot's exact d2 to the union

    def knn_select(self, x, knn, measure, p0, p1):
        from .graph import knn_select_device

        return knn_select_device(x, knn, measure, p0, p1, with_vals=True)

    def knn_union(self, x, knn, measure, sel, perm, r0, r1, sel_vals=None):
        from .graph import knn_union_device

        return knn_union_device(x, knn, measure, sel, perm, r0, r1, sel_vals)

    def is_symmetric(self, w: DeviceCsr) -> bool:
        from .sparse import is_symmetric

        return is_symmetric(w)

    def slice_rows(self, w: DeviceCsr, r0: int, r1: int) -> DeviceCsr:
        rp = w.row_ptr[r0 : r1 + 1]
        b, e = int(rp[0].item()), int(rp[-1].item())
        return DeviceCsr(r1 - r0, w.n_cols, (rp - b).contiguous(), w.col[b:e], w.vals[b:e])

    def degrees(self, a: DeviceCsr):
        from .laplacian import degrees_device

        return degrees_device(a)

    def zeros_count(self, d) -> int:
        from .laplacian import nonpositive_device

        return nonpositive_device(d, 0)[0]

    def sym_scale_shard(self, a: DeviceCsr, r0: int, d_full):
        out = self.torch.empty_like(a.vals)
        nat.check(self.lib.sc_sym_scale_shard_f64(a.n_rows, r0, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals),
                                                  nat.ptr(d_full), nat.ptr(out), self._s()))
        return a.with_vals(out)

    # ---- Lanczos blocks (basis: tensor (m+1, ld); row c = basis vector c)
    def spmv(self, a: DeviceCsr, x_full):
        y = self.torch.empty(a.n_rows, dtype=self.torch.float64, device="cuda")
        nat.check(self.lib.sc_spmv_f64(a.n_rows, a.n_cols, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals),
                                       nat.ptr(x_full), nat.ptr(y), 0, self._s()))
        return y

    def operator(self, a: DeviceCsr):
        """Repeated y = A_local x_full: the CSR warp-per-row kernel, or a
        SELL-32-sigma handle when SPECLUST_SPMV_FORMAT=sell (as in the
        single-GPU eigensolver)."""
        import os

        if os.environ.get("SPECLUST_SPMV_FORMAT") == "sell":
            return _SellOp(self, a)
        return _CsrOp(self, a)

    def gemv_t(self, B, ncols, w):
        h = self.torch.empty(max(1, ncols), dtype=self.torch.float64, device="cuda")
        nat.check(self.lib.sc_gemv_t_f64(w.numel(), B.shape[1], ncols, nat.ptr(B), nat.ptr(w), nat.ptr(h), self._s()))
        return h[:ncols]

    def gemv_n(self, B, ncols, h, w, want_sq=False):
        sq = self.torch.zeros(1, dtype=self.torch.float64, device="cuda") if want_sq else None
        nat.check(self.lib.sc_gemv_n_f64(w.numel(), B.shape[1], ncols, nat.ptr(B), nat.ptr(h), nat.ptr(w),
                                         nat.ptr(sq), self._s()))
        return sq

    def div_into(self, dst, src, div):
        nat.check(self.lib.sc_div_copy_f64(src.numel(), nat.ptr(src), float(div), nat.ptr(dst), self._s()))

    def normal(self, n, offset, seed, stream_id):
        out = self.torch.empty(n, dtype=self.torch.float64, device="cuda")
        nat.check(self.lib.sc_fill_normal(n, offset, seed & (2**64 - 1), stream_id, nat.ptr(out), self._s()))
        return out

    def symeig(self, T: np.ndarray, k: int, p=None):
        """(theta host (m,) stable descending, S device (k, m): row c =
        eigenvector c).  With p: T's rows 0..p-1 are diag(theta) coupled only
        to row p (the thick restart's arrowhead), the rest tridiagonal -- the
        arrowhead divide and conquer of the single-GPU solver; p=None: any
        dense symmetric T (Householder + QL)."""
        m = T.shape[0]
        Td = nat.to_device(np.asfortranarray(T).ravel(order="F"), self.torch.float64)
        theta = self.torch.empty(m, dtype=self.torch.float64, device="cuda")
        S = self.torch.empty((k, m), dtype=self.torch.float64, device="cuda")
        if p is None:
            nat.check(self.lib.sc_symeig_f64(m, k, nat.ptr(Td), nat.ptr(theta), nat.ptr(S), self._s()))
        else:
            nat.check(self.lib.sc_symeig_arrow_f64(m, p, k, nat.ptr(Td), nat.ptr(theta), nat.ptr(S), self._s()))
        return nat.to_host(theta), S

    def ritz(self, B, nl, m, S, k, rowmajor=False):
        """B[:m] combined by S: col-major (k, ld) tensor or row-major (nl, k)."""
        ld = B.shape[1]
        if rowmajor:
            out = self.torch.empty((nl, k), dtype=self.torch.float64, device="cuda")
            ldc = k
        else:
            out = self.torch.empty((k, ld), dtype=self.torch.float64, device="cuda")
            ldc = ld
        nat.check(self.lib.sc_dgemm_tall(nl, m, k, nat.ptr(B), ld, nat.ptr(S), m, nat.ptr(out), ldc,
                                         1 if rowmajor else 0, self._s()))
        return out

    # ---- embedding
    def embed_scale(self, U, d_local):
        V = self.torch.empty_like(U)
        colsq = self.torch.zeros(U.shape[1], dtype=self.torch.float64, device="cuda")
        nat.check(self.lib.sc_embed_scale(U.shape[0], U.shape[1], nat.ptr(U), nat.ptr(d_local), nat.ptr(V),
                                          nat.ptr(colsq), self._s()))
        return V, colsq

    def embed_finish(self, V, colsq, normalize_rows):
        nat.check(self.lib.sc_embed_finish(V.shape[0], V.shape[1], nat.ptr(colsq), 1 if normalize_rows else 0,
                                           nat.ptr(V), self._s()))
        return V

    # ---- k-means blocks
    def kmeans_assign(self, V, C, old):
        n = V.shape[0]
        labels = self.torch.empty(n, dtype=self.torch.int64, device="cuda")
        cost = self.torch.empty(n, dtype=self.torch.float64, device="cuda")
        chg, sse = nat.C.c_int64(0), nat.C.c_double(0.0)
        nat.check(self.lib.sc_kmeans_assign(n, V.shape[1], C.shape[0], nat.ptr(V), nat.ptr(C), nat.ptr(old),
                                            nat.ptr(labels), nat.ptr(cost), nat.C.byref(chg), nat.C.byref(sse),
                                            self._s()))
        return labels, cost, int(chg.value), float(sse.value)

    def local_sums(self, V, labels, k):
        d = V.shape[1]
        sums = self.torch.empty((k, d), dtype=self.torch.float64, device="cuda")
        counts = self.torch.empty(k, dtype=self.torch.int64, device="cuda")
        nat.check(self.lib.sc_kmeans_local_sums(V.shape[0], d, k, nat.ptr(V), nat.ptr(labels), nat.ptr(sums),
                                                nat.ptr(counts), self._s()))
        return sums, counts

    def divide(self, sums, counts):
        C = self.torch.empty_like(sums)
        nat.check(self.lib.sc_centroid_divide(sums.shape[0], sums.shape[1], nat.ptr(sums), nat.ptr(counts),
                                              nat.ptr(C), self._s()))
        return C

    def farthest(self, cost_full, e):
        idx = np.zeros(max(1, e), dtype=np.int64)
        nat.check(self.lib.sc_farthest(cost_full.numel(), nat.ptr(cost_full), e,
                                       idx.ctypes.data_as(nat.P_i64), self._s()))
        return idx[:e]

    def kpp_session(self, V):
        return _CudaKpp(self, V)

    def ncut_partials(self, a: DeviceCsr, r0, labels_full, k):
        bnd = self.torch.empty(k, dtype=self.torch.float64, device="cuda")
        vol = self.torch.empty(k, dtype=self.torch.float64, device="cuda")
        cnt = self.torch.empty(k, dtype=self.torch.int64, device="cuda")
        nat.check(self.lib.sc_ncut_partials(a.n_rows, r0, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals),
                                            nat.ptr(labels_full), k, nat.ptr(bnd), nat.ptr(vol), nat.ptr(cnt),
                                            self._s()))
        return bnd, vol, cnt


class _CsrOp:
    """sc_spmv_plan_* handle of a row-shard operator (rows local, columns
    global): built once, applied per Lanczos step without host syncs."""

    def __init__(self, ops: CudaOps, a: DeviceCsr):
        self.ops, self.a = ops, a  # keeps the CSR arrays alive with the handle
        self.h = nat.vp()
        nat.check(ops.lib.sc_spmv_plan_create(a.n_rows, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals),
                                              ops._s(), nat.C.byref(self.h)))

    def apply(self, x_full):
        y = self.ops.torch.empty(self.a.n_rows, dtype=self.ops.torch.float64, device="cuda")
        nat.check(self.ops.lib.sc_spmv_plan_apply(self.h, nat.ptr(x_full), nat.ptr(y), self.ops._s()))
        return y

    def close(self):
        if self.h:
            self.ops.lib.sc_spmv_plan_destroy(self.h)
            self.h = nat.vp()


class _SellOp:
    """sc_sell_* handle of a row-shard operator (rows local, columns global)."""

    def __init__(self, ops: CudaOps, a: DeviceCsr):
        self.ops, self.a = ops, a  # keeps the CSR arrays alive with the handle
        self.h = nat.vp()
        nat.check(ops.lib.sc_sell_create(a.n_rows, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), ops._s(),
                                         nat.C.byref(self.h)))

    def apply(self, x_full):
        y = self.ops.torch.empty(self.a.n_rows, dtype=self.ops.torch.float64, device="cuda")
        nat.check(self.ops.lib.sc_sell_spmv(self.h, nat.ptr(x_full), nat.ptr(y), self.ops._s()))
        return y

    def close(self):
        if self.h is not None and self.h.value:
            self.ops.lib.sc_sell_destroy(self.h)
            self.h = None


class _CudaKpp:
    """Shard view of the device k-means++ state (sc_kmeanspp_*)."""

    def __init__(self, ops: CudaOps, V):
        self.ops, self.V = ops, V
        self.h = nat.vp()
        nat.check(ops.lib.sc_kmeanspp_create(V.shape[0], V.shape[1], nat.ptr(V), ops._s(), nat.C.byref(self.h)))

    def close(self):
        if self.h is not None and self.h.value:
            self.ops.lib.sc_kmeanspp_destroy(self.h)
            self.h = None

    def take_row(self, row, local_index):
        nat.check(self.ops.lib.sc_kmeanspp_take_row(self.h, nat.ptr(row), int(local_index)))

    def weight(self):
        w, c, f = nat.C.c_double(0.0), nat.C.c_int64(0), nat.C.c_int64(0)
        nat.check(self.ops.lib.sc_kmeanspp_weight(self.h, nat.C.byref(w), nat.C.byref(c), nat.C.byref(f)))
        return float(w.value), int(c.value), int(f.value)

    def psum(self, total):
        p = nat.C.c_double(0.0)
        nat.check(self.ops.lib.sc_kmeanspp_psum(self.h, float(total), nat.C.byref(p)))
        return float(p.value)

    def search(self, target):
        i = nat.C.c_int64(-1)
        nat.check(self.ops.lib.sc_kmeanspp_search(self.h, float(target), nat.C.byref(i)))
        return int(i.value)

    def nth_free(self, r):
        i = nat.C.c_int64(-1)
        nat.check(self.ops.lib.sc_kmeanspp_nth_free(self.h, int(r), nat.C.byref(i)))
        return int(i.value)


# ---------------------------------------------------------------------------
# query-sharded kNN graph (graph.py:185-237)
def scan_bounds(n: int, world: int) -> list[int]:
    """Scan-position shards in whole 128-point query tiles."""
    tiles = -(-n // 128)
    return [min(n, b * 128) for b in row_bounds(tiles, world)]


def knn_graph_sharded(ops, comm: Comm, x, knn: int, measure):
    """Row block [bounds[rank], bounds[rank+1]) of the union-kNN graph.

    Each rank selects the top-knn of its query tiles (the tensor-core scan
    against all points), one all-gather assembles the n x knn selection (the
    exchange that carries the reverse edges), and each rank emits its own CSR
    rows from it.  Returns (local CSR, row bounds)."""
    xd = ops.points(x)
    n = int(xd.shape[0])
    pb = scan_bounds(n, comm.world)
    bounds = row_bounds(n, comm.world)
    if getattr(ops, "carries_vals", False):
        # the value-carrying union (as on one GPU): the exact d2 of every
        # selection slot travels with the selection, so no rank recomputes
        # distances for its reverse edges
        sel_loc, perm, vals_loc = ops.knn_select(xd, knn, measure, pb[comm.rank], pb[comm.rank + 1])
        sel = comm.gather_rows(sel_loc.contiguous(), pb)
        sel_vals = comm.gather_rows(vals_loc.contiguous(), pb)
        w_loc = ops.knn_union(xd, knn, measure, sel, perm, bounds[comm.rank], bounds[comm.rank + 1], sel_vals)
        return w_loc, bounds
    sel_loc, perm = ops.knn_select(xd, knn, measure, pb[comm.rank], pb[comm.rank + 1])
    sel = comm.gather_rows(sel_loc.contiguous(), pb)
    w_loc = ops.knn_union(xd, knn, measure, sel, perm, bounds[comm.rank], bounds[comm.rank + 1])
    return w_loc, bounds


def knn_graph_sharded_full(ops, comm: Comm, x, knn: int, measure):
    """Like knn_graph_sharded, but every rank emits the WHOLE union from the
    gathered selection (O(nnz) replicated work; the O(N^2 d) candidate scan
    stays sharded), so the eigensolver can run on the locality-ordered
    operator P A P^T in scan-order row blocks, as on one GPU.  Returns (W,
    perm)."""
    xd = ops.points(x)
    n = int(xd.shape[0])
    pb = scan_bounds(n, comm.world)
    sel_loc, perm, vals_loc = ops.knn_select(xd, knn, measure, pb[comm.rank], pb[comm.rank + 1])
    sel = comm.gather_rows(sel_loc.contiguous(), pb)
    sel_vals = comm.gather_rows(vals_loc.contiguous(), pb)
    return ops.knn_union(xd, knn, measure, sel, perm, 0, n, sel_vals), perm


# ---------------------------------------------------------------------------
# row-sharded thick-restart Lanczos (eigen.py:86-302)
def _deflate_min_n() -> int:
    return int(os.environ.get("SPECLUST_DEFLATE_MIN_N", "32768"))


class _LockedShards:
    """The eigenvalue-1 eigenvectors of A = D^-1/2 W D^-1/2, one per
    connected component (u_C = D^1/2 1_C / |D^1/2 1_C|, disjoint supports),
    row-sharded like the operator: the sharded counterpart of
    sc_eigensolve_csr_deflate.  Components by min-label propagation with
    one pointer jump per pass over the local rows and an all-gather of the
    labels; per-component sums by a stable sort of the local rows by
    component (segment_reduce: fixed order) and one all-reduce of c values."""

    def __init__(self, comm, a_local, bounds, d_local):
        torch = comm.torch
        self.comm, self.torch = comm, torch
        r0, r1 = bounds[comm.rank], bounds[comm.rank + 1]
        n = bounds[-1]
        dev = d_local.device
        rp = a_local.row_ptr.to(dev, torch.int64)
        cols = a_local.col.to(dev, torch.int64)
        rows = torch.repeat_interleave(torch.arange(r1 - r0, device=dev), torch.diff(rp))
        lab = torch.arange(n, device=dev, dtype=torch.int64)
        for _ in range(100000):
            loc = lab[r0:r1].clone()
            if cols.numel():
                loc.scatter_reduce_(0, rows, lab[cols], reduce="amin")
            new = comm.gather_rows(loc, bounds)
            new = torch.minimum(new, new[new])  # one pointer jump
            changed = torch.tensor([float((new != lab).any().item())], dtype=torch.float64, device=dev)
            lab = new
            if comm.sum_(changed)[0].item() == 0.0:
                break
        roots = lab == torch.arange(n, device=dev, dtype=torch.int64)
        rank = torch.cumsum(roots.to(torch.int64), 0) - 1
        self.c = int(roots.sum().item())
        self.comp = rank[lab[r0:r1]]  # local rows -> component id (ordered by smallest node)
        self.order = torch.sort(self.comp, stable=True).indices
        self.lengths = torch.bincount(self.comp, minlength=self.c)
        dsum = self.seg_sum(d_local)
        self.u = torch.sqrt(d_local) / torch.sqrt(dsum[self.comp])

    def seg_sum(self, v):
        """sum of v over each component's rows on every rank (length c)"""
        out = self.torch.segment_reduce(v[self.order], "sum", lengths=self.lengths)
        return self.comm.sum_(out.contiguous())

    def deflate(self, v):
        h = self.seg_sum(self.u * v)
        v -= h[self.comp] * self.u
        return v


def lanczos_sharded(ops, comm: Comm, a_local, n: int, bounds, cfg: LanczosConfig, d_local=None):
    """Top-k eigenpairs of the symmetric operator whose row block
    [bounds[rank], bounds[rank+1]) is ``a_local`` (global column indices).

    Returns (values host (k,), vectors local (nl, k) row-major, residuals host
    (k,), stats dict).  Raises MaxRestartsExceeded / Breakdown like eigen.py."""
    op = ops.operator(a_local) if hasattr(ops, "operator") else None
    try:
        if d_local is not None and n >= _deflate_min_n() and cfg.k >= 2 and \
                os.environ.get("SPECLUST_DEFLATE", "1") != "0":
            return _lanczos_sharded_deflate(ops, comm, a_local, n, bounds, cfg, op, d_local)
        return _lanczos_sharded(ops, comm, a_local, n, bounds, cfg, op)
    finally:
        if op is not None:
            op.close()


def _lanczos_sharded_deflate(ops, comm, a_local, n, bounds, cfg, op, d_local):
    """A = D^-1/2 W D^-1/2 with 2 <= c < k connected components: the c
    eigenvalue-1 pairs locked (_LockedShards), the Lanczos recurrence for the
    other k - c on their orthogonal complement (subspace m - c); else the
    plain sharded solve.  stats["locked"] = c."""
    torch = comm.torch
    k = cfg.k
    m = cfg.m if cfg.m is not None else default_subspace_dim(n, k)
    lk = _LockedShards(comm, a_local, bounds, d_local)
    c = lk.c
    if not 2 <= c < k:
        return _lanczos_sharded(ops, comm, a_local, n, bounds, cfg, op)

    def matvec(x_full):
        return op.apply(x_full) if op is not None else ops.spmv(a_local, x_full)

    y = matvec(comm.gather_rows(lk.u.contiguous(), bounds))
    theta_l = lk.seg_sum(lk.u * y)
    res_l = torch.sqrt(lk.seg_sum((y - theta_l[lk.comp] * lk.u) ** 2))
    th, rs = ops.host(theta_l), ops.host(res_l)
    if not (np.all(np.abs(th - 1.0) <= 1e-10) and np.all(rs <= 1e-3 * float(cfg.tol))):
        return _lanczos_sharded(ops, comm, a_local, n, bounds, cfg, op)
    sub = LanczosConfig(k=k - c, m=m - c, tol=cfg.tol, max_restarts=cfg.max_restarts, seed=cfg.seed)
    values, V, residuals, st = _lanczos_sharded(ops, comm, a_local, n, bounds, sub, op, deflate=lk.deflate)
    ordr = np.argsort(-th, kind="stable")
    col_of = np.empty(c, dtype=np.int64)
    col_of[ordr] = np.arange(c)
    nl = bounds[comm.rank + 1] - bounds[comm.rank]
    out = ops.zeros((nl, k))
    if nl:
        cols = torch.as_tensor(col_of, device=lk.u.device)[lk.comp]
        out[torch.arange(nl, device=lk.u.device), cols] = lk.u
        out[:, c:] = V
    st["locked"] = c
    st["m"] = m
    return (np.concatenate([th[ordr], values]), out, np.concatenate([rs[ordr], residuals]), st)


def _lanczos_sharded(ops, comm, a_local, n, bounds, cfg, op, deflate=None):
    def matvec(x_full):
        w = op.apply(x_full) if op is not None else ops.spmv(a_local, x_full)
        return deflate(w) if deflate is not None else w

    k = cfg.k
    m = cfg.m if cfg.m is not None else default_subspace_dim(n, k)
    if not (1 <= k < m <= n):
        raise BadConfig(f"need 1 <= k < m <= n, got k={k}, m={m}, n={n}")
    if not cfg.tol > 0:
        raise BadConfig(f"tol must be positive, got {cfg.tol}")
    r0, r1 = bounds[comm.rank], bounds[comm.rank + 1]
    nl = r1 - r0
    seed = int(cfg.seed) & (2**64 - 1)
    tol = float(cfg.tol)
    B = ops.zeros((m + 1, max(nl, 1)))
    T = np.zeros((m, m))
    st = dict(restarts=0, breakdowns=0, matvecs=0, history=[], m=m)
    rng_stream = [0]

    def dot_all(h):
        return comm.sum_(h)

    def norm_of(v):
        sq = ops.gemv_n(B, 0, None, v, want_sq=True)
        return math.sqrt(float(comm.sum_(sq)[0].item()))

    def cgs2(v, count):
        if count == 0:
            return norm_of(v)
        h = dot_all(ops.gemv_t(B, count, v))
        ops.gemv_n(B, count, h, v)
        h = dot_all(ops.gemv_t(B, count, v))
        sq = ops.gemv_n(B, count, h, v, want_sq=True)
        return math.sqrt(float(comm.sum_(sq)[0].item()))

    def fresh(count, dst, is_breakdown):
        for _ in range(3):
            rng_stream[0] += 1
            v = ops.normal(nl, r0, seed, rng_stream[0])
            if deflate is not None:
                deflate(deflate(v))
            nv = cgs2(v, count)
            if nv > 1e-6 * math.sqrt(n):
                if is_breakdown:
                    st["breakdowns"] += 1
                ops.div_into(B[dst, :nl], v, nv)
                return
        raise Breakdown(f"could not extend the basis past {count} vectors")

    v0 = ops.normal(nl, r0, seed, 0)
    if deflate is not None:
        deflate(deflate(v0))
    ops.div_into(B[0, :nl], v0, norm_of(v0))
    scale = 0.0
    pending = None
    j = 0
    st["second_passes"] = 0
    while True:
        x_full = comm.gather_rows(B[j, :nl].contiguous(), bounds)
        w = matvec(x_full)
        st["matvecs"] += 1
        cnt = j + 1
        # one full CGS pass (subsumes the three-term recurrence, eigen.py:157-163)
        # and a second only when the first cancelled most of |w| (DGKS; the
        # same rule as the single-GPU session, sc_lanczos.cu advance())
        # [B^T w; |w|^2] in ONE all-reduce, |w - B h|^2 in a second, and one
        # host read of (alpha, |w|^2, beta^2) per step
        torch = comm.torch
        hs = torch.cat([ops.gemv_t(B, cnt, w), ops.gemv_n(B, 0, None, w, want_sq=True)])
        comm.sum_(hs)
        sq = ops.gemv_n(B, cnt, hs[:cnt], w, want_sq=True)
        comm.sum_(sq)
        alpha, w0sq, bsq = (float(v) for v in ops.host(torch.stack([hs[j], hs[cnt], sq[0]])))
        T[j, j] = alpha
        beta = math.sqrt(bsq)
        if beta < REORTH_ETA * math.sqrt(w0sq):
            st["second_passes"] += 1
            h = dot_all(ops.gemv_t(B, cnt, w))
            sq = ops.gemv_n(B, cnt, h, w, want_sq=True)
            beta = math.sqrt(float(ops.host(comm.sum_(sq))[0]))
        scale = max(scale, abs(alpha), beta)
        if j + 1 < m:
            if beta > BREAKDOWN_RTOL * max(1.0, scale):
                T[j, j + 1] = T[j + 1, j] = beta
                ops.div_into(B[j + 1, :nl], w, beta)
            else:
                T[j, j + 1] = T[j + 1, j] = 0.0
                fresh(j + 1, j + 1, True)
            j += 1
            continue
        # ---- sweep complete (eigen.py:187-239), replicated on every rank
        theta, S = ops.symeig(T, k, k if st["restarts"] > 0 else 0)
        last = ops.host(S[:, m - 1])
        est = beta * np.abs(last)
        st["history"].append(float(est.max()))
        # the single-GPU session's margin (sc_lanczos.cu kConvMargin: 4x below
        # 32768 rows, the reference's own test above)
        margin = 1.0 if n >= 32768 else 0.25
        converged = bool(np.all(est <= margin * tol * np.maximum(1.0, np.abs(theta[:k]))))
        verified = False
        if pending is not None:
            slack = np.maximum(1.0, np.abs(theta[:k])) * max(tol, 1e-12)
            verified = bool(np.all(np.abs(theta[:k] - pending) <= slack))
        if converged and (m == n or verified):
            V = ops.ritz(B, nl, m, S, k, rowmajor=True)  # (nl, k)
            # unit columns (eigen.py:204): global column norms via the
            # embedding blocks with unit degrees
            V, colsq = ops.embed_scale(V, ops.ones(nl))
            comm.sum_(colsq)
            V = ops.embed_finish(V, colsq, False)
            values = theta[:k].copy()
            res = np.zeros(k)
            one = ops.zeros((1,))
            for i in range(k):  # true residuals |A v - theta v| (eigen.py:241-248)
                vi = V[:, i].contiguous()
                xg = comm.gather_rows(vi, bounds)
                yi = op.apply(xg) if op is not None else ops.spmv(a_local, xg)
                one.fill_(values[i])
                sq = ops.gemv_n(vi.reshape(1, -1), 1, one, yi, want_sq=True)
                res[i] = float(comm.sum_(sq)[0].item())
            return values, V, np.sqrt(res), st
        if st["restarts"] >= cfg.max_restarts:
            raise MaxRestartsExceeded(f"{st['restarts']} restarts without verified convergence; worst residual "
                                      f"estimate {est.max():.3e}", values=theta[:k].copy(), residuals=est)
        st["restarts"] += 1
        Y = ops.ritz(B, nl, m, S, k)  # (k, ld)
        B[:k] = Y
        coupled = (not converged) and beta > BREAKDOWN_RTOL * max(1.0, scale)
        T[:] = 0.0
        T[np.arange(k), np.arange(k)] = theta[:k]
        if converged:
            pending = theta[:k].copy()
            fresh(k, k, False)
        else:
            pending = None
            if coupled:
                T[:k, k] = T[k, :k] = beta * last
                ops.div_into(B[k, :nl], w, beta)
            else:
                fresh(k, k, True)
        j = k


# ---------------------------------------------------------------------------
# point-sharded k-means++ and Lloyd (kmeans.py:107-196)
def _owner(bounds, g):
    return int(np.searchsorted(np.asarray(bounds), g, side="right") - 1)


def _row_of(ops, comm, V, bounds, g):
    """Coordinates of global row g, broadcast from its owner."""
    owner = _owner(bounds, g)
    row = ops.zeros((V.shape[1],))
    if comm.rank == owner:
        row.copy_(V[g - bounds[owner]])
    return comm.bcast_(row, owner)


def kmeanspp_sharded(ops, comm: Comm, V, bounds, k: int, seed):
    """Global row indices chosen by k-means++ with the reference's numpy draws."""
    n = bounds[-1]
    if not 1 <= k <= n:
        raise BadConfig(f"k must satisfy 1 <= k <= n, got k={k}, n={n}")
    r0 = bounds[comm.rank]
    rng = np.random.default_rng(seed)
    sess = ops.kpp_session(V)
    try:
        chosen = np.empty(k, dtype=np.int64)
        chosen[0] = rng.integers(n)
        g = int(chosen[0])
        sess.take_row(_row_of(ops, comm, V, bounds, g), g - r0 if bounds[comm.rank] <= g < bounds[comm.rank + 1] else -1)
        for i in range(1, k):
            w, c, f = sess.weight()
            tab = comm.gather_scalars([w, c, f])  # (world, 3)
            counts = tab[:, 1].astype(np.int64)
            if counts.sum() > 0:
                total = float(tab[:, 0].sum())
                u = rng.random()  # Generator.choice(len, p=...) draws one double
                ps = comm.gather_scalars([sess.psum(total)])[:, 0]
                target = u * float(ps.sum())
                prefix = np.concatenate(([0.0], np.cumsum(ps)))
                owner = int(np.argmax(prefix[1:] > target)) if np.any(prefix[1:] > target) else \
                    int(np.flatnonzero(counts)[-1])
                loc = sess.search(target - prefix[owner]) if comm.rank == owner else -1
                pick = comm.gather_scalars([loc])[owner, 0]
                g = int(pick) + bounds[owner]
            else:
                frees = tab[:, 2].astype(np.int64)
                r = int(rng.integers(int(frees.sum())))
                fpre = np.concatenate(([0], np.cumsum(frees)))
                owner = int(np.searchsorted(fpre, r, side="right") - 1)
                loc = sess.nth_free(r - fpre[owner]) if comm.rank == owner else -1
                g = int(comm.gather_scalars([loc])[owner, 0]) + bounds[owner]
            chosen[i] = g
            mine = bounds[comm.rank] <= g < bounds[comm.rank + 1]
            sess.take_row(_row_of(ops, comm, V, bounds, g), g - r0 if mine else -1)
        return chosen
    finally:
        sess.close()


def lloyd_sharded(ops, comm: Comm, V, bounds, init_c, cfg: KmeansConfig):
    """Lloyd iterations on point shards; returns (labels local, centroids,
    sse_history host, iters)."""
    k = init_c.shape[0]
    labels, cost, _, sse = ops.kmeans_assign(V, init_c, None)
    hist = [float(comm.gather_scalars([sse])[:, 0].sum())]
    C = init_c
    it = 0
    while it < cfg.max_iters:
        sums, counts = ops.local_sums(V, labels, k)
        comm.sum_(sums)
        comm.sum_(counts)
        C = ops.divide(sums, counts)
        hc = ops.host(counts)
        empties = np.flatnonzero(hc == 0)
        if len(empties):  # kmeans.py:149-155, over all shards
            cost_full = comm.gather_rows(cost, bounds)
            far = ops.farthest(cost_full, len(empties))
            for slot, cl in enumerate(empties):
                C[cl] = _row_of(ops, comm, V, bounds, int(far[slot]))
        new, cost, chg, sse = ops.kmeans_assign(V, C, labels)
        tab = comm.gather_scalars([chg, sse])
        hist.append(float(tab[:, 1].sum()))
        it += 1
        labels = new
        if int(tab[:, 0].sum()) <= cfg.tol_changes:
            break
    return labels, C, np.array(hist), it


def kmeans_sharded(ops, comm, V, bounds, cfg: KmeansConfig):
    n = bounds[-1]
    if cfg.k > n:
        raise BadConfig(f"k={cfg.k} exceeds number of points n={n}")
    best = None
    for r in range(cfg.restarts):
        seed = cfg.seed if r == 0 else int(np.random.SeedSequence([cfg.seed, r]).generate_state(1)[0])
        if cfg.init == "kmeanspp":
            rows = kmeanspp_sharded(ops, comm, V, bounds, cfg.k, seed)
        else:
            rows = np.random.default_rng(seed).choice(n, size=cfg.k, replace=False)
        init_c = ops.zeros((cfg.k, V.shape[1]))
        for i, g in enumerate(rows):
            init_c[i] = _row_of(ops, comm, V, bounds, int(g))
        cand = lloyd_sharded(ops, comm, V, bounds, init_c, cfg)
        if best is None or cand[2][-1] < best[2][-1]:
            best = cand
    return best


# ---------------------------------------------------------------------------
@dataclass
class ShardedResult:
    report: object
    bounds: list


def run_sharded(cfg, comm: Comm, ops=None):
    """run() with the eigen and k-means stages sharded over ``comm``.

    Every rank returns the same ClusterReport (labels of all points)."""
    import time

    from .graph import as_points
    from .pipeline import ClusterReport, MatrixInput, PointsInput

    ops = ops or CudaOps()
    torch = ops.torch
    timings = {}
    warnings: list[str] = []

    def sync():
        if ops.device == "cuda":
            torch.cuda.synchronize()

    t = time.perf_counter()
    src = cfg.input
    # locality-ordered eigensolve (the single-GPU pipeline's P A P^T in scan
    # order) whenever the ops carry the selection's values (CUDA shards)
    locality = isinstance(src, PointsInput) and src.pattern == "knn" and getattr(ops, "carries_vals", False)
    if isinstance(src, PointsInput) and src.pattern == "knn":
        pts = src.points if isinstance(src.points, torch.Tensor) else as_points(src.points)
        if src.measure.kind != "exp_decay":
            raise NotImplementedError("the sharded kNN graph supports the exp_decay measure")
        if locality:
            w_full, perm = knn_graph_sharded_full(ops, comm, pts, src.knn, src.measure)
            n = w_full.n_rows
            bounds = row_bounds(n, comm.world)
            w_loc = ops.slice_rows(w_full, bounds[comm.rank], bounds[comm.rank + 1])
        else:
            w_loc, bounds = knn_graph_sharded(ops, comm, pts, src.knn, src.measure)
            n = bounds[-1]
    elif isinstance(src, MatrixInput) and src.matrix is not None:
        from .sparse import CsrMatrix, coo_canonicalize, coo_to_csr

        m = src.matrix
        host = m if isinstance(m, CsrMatrix) else coo_to_csr(coo_canonicalize(m))
        w = ops.from_host_csr(host) if hasattr(ops, "from_host_csr") else host.device()
        n = w.n_rows
        # the reference's _resolve_graph gates (pipeline.py:181-192): exact
        # symmetry (every rank holds the whole matrix here) and the
        # negative-weight warning
        if not ops.is_symmetric(w):
            raise NotSymmetric("similarity matrix must be symmetric")
        if host.nnz and host.vals.min() < 0.0:
            warnings.append("similarity matrix contains negative weights")
        bounds = row_bounds(n, comm.world)
        w_loc = ops.slice_rows(w, bounds[comm.rank], bounds[comm.rank + 1])
        del w
    else:
        raise NotImplementedError("sharded run supports PointsInput(pattern='knn') and in-memory MatrixInput")
    r0, r1 = bounds[comm.rank], bounds[comm.rank + 1]
    sync()
    timings["graph"] = time.perf_counter() - t

    t = time.perf_counter()
    if locality:  # replicated: every rank holds the whole W
        d_full = ops.degrees(w_full)
        d_loc = d_full[r0:r1]
        zeros = ops.zeros_count(d_full)
    else:
        d_loc = ops.degrees(w_loc)
        zeros = int(comm.gather_scalars([ops.zeros_count(d_loc)])[:, 0].sum())
        d_full = comm.gather_rows(d_loc, bounds)
    if zeros:
        if cfg.isolated_policy == "error":
            idx = np.flatnonzero(ops.host(d_full) == 0.0)
            raise IsolatedNode(idx)
        raise NotImplementedError("isolated_policy='remove' is not sharded yet")
    if n < cfg.k_clusters:
        raise BadConfig(f"graph has {n} usable nodes but k_clusters={cfg.k_clusters}")
    sync()
    timings["degrees"] = time.perf_counter() - t

    t = time.perf_counter()
    ecfg = cfg.eigen if cfg.eigen is not None else LanczosConfig(k=cfg.k_clusters)
    if locality:
        from .pipeline import permute_device

        a_p, pos = permute_device(ops.sym_scale_shard(w_full, 0, d_full), perm)
        a_loc = ops.slice_rows(a_p, r0, r1)  # scan positions [r0, r1)
        del a_p
    else:
        a_loc = ops.sym_scale_shard(w_loc, r0, d_full)
    # degrees in the operator's row order (scan order on the locality path)
    d_op = d_full[perm.to(d_full.device, torch.int64)][r0:r1] if locality else d_loc
    try:
        values, U, residuals, est = lanczos_sharded(ops, comm, a_loc, n, bounds, ecfg, d_local=d_op.contiguous())
    except MaxRestartsExceeded as e:
        raise EigenNotConverged(e) from e
    if locality:
        # the eigenvector rows back to point order (the k-means++ draws index
        # points): scan position r0 + i holds point perm[r0 + i]
        pts_ids = perm[r0:r1].to(torch.int64)
        bt = torch.tensor(bounds, dtype=torch.int64, device=pts_ids.device)
        owner = torch.searchsorted(bt, pts_ids, right=True) - 1
        U = comm.exchange_rows(U.contiguous(), owner, pts_ids - bt[owner], r1 - r0)
    V, colsq = ops.embed_scale(U, d_loc)
    comm.sum_(colsq)
    V = ops.embed_finish(V, colsq, cfg.normalize_rows)
    sync()
    timings["eigen"] = time.perf_counter() - t

    t = time.perf_counter()
    kcfg = cfg.kmeans if cfg.kmeans is not None else KmeansConfig(k=cfg.k_clusters)
    labels_loc, C, hist, iters = kmeans_sharded(ops, comm, V, bounds, kcfg)
    sync()
    timings["kmeans"] = time.perf_counter() - t

    t = time.perf_counter()
    labels_full = comm.gather_rows(labels_loc, bounds)
    bnd, vol, cnt = ops.ncut_partials(w_loc, r0, labels_full, kcfg.k)
    comm.sum_(bnd)
    comm.sum_(vol)
    comm.sum_(cnt)
    hb, hv, hc = ops.host(bnd), ops.host(vol), ops.host(cnt)
    occ = hc > 0
    if np.any(hv[occ] <= 0.0):
        raise ZeroVolumePart("a part has zero volume")
    ncut_value = 0.5 * float((hb[occ] / hv[occ]).sum())
    if int(occ.sum()) < cfg.k_clusters:
        warnings.append(f"clustering occupies {int(occ.sum())} of {cfg.k_clusters} clusters")
    labels = ops.host(labels_full)
    sync()
    timings["metrics"] = time.perf_counter() - t

    lab = Labeling(labels, ops.host(C), float(hist[-1]), iters, hist)
    last_info.clear()
    last_info["nnz"] = int(comm.gather_scalars([w_loc.nnz])[:, 0].sum())
    last_info["eigen"] = dict(est, world=comm.world, locality_order=locality)
    rep = ClusterReport(labeling=lab, eigenvalues=nat.frozen(values), eigen_residuals=nat.frozen(residuals),
                        ncut_value=ncut_value, timings=timings, warnings=warnings,
                        index_map=np.arange(n, dtype=np.int64))
    return rep
