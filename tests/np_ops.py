"""Numpy implementation of the per-shard ops interface of
paper_1802_04450_b200.distributed — TEST INFRASTRUCTURE ONLY.

It lets the sharded drivers (row-sharded Lanczos, point-sharded k-means,
sharded pipeline) run on CPU tensors under a gloo process group, so their
distributed logic is covered without GPUs.  Numerics follow the CPU oracle.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import speclust_oracle as orc


class HostCsr:
    def __init__(self, n_rows, n_cols, row_ptr, col, vals):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr, self.col, self.vals = row_ptr, col, vals

    @property
    def nnz(self):
        return int(self.col.numel())

    def with_vals(self, vals):
        return HostCsr(self.n_rows, self.n_cols, self.row_ptr, self.col, vals)


def _t(a, dtype=torch.float64):
    return torch.from_numpy(np.array(a, copy=True)).to(dtype)


class NumpyOps:
    device = "cpu"
    torch = torch

    def zeros(self, shape, dtype=None):
        return torch.zeros(shape, dtype=dtype or torch.float64)

    def ones(self, n):
        return torch.ones(n, dtype=torch.float64)

    def host(self, t):
        return t.detach().cpu().numpy().copy()

    # ---- graph / normalisation
    def knn_graph(self, x, knn, measure):
        x = np.asarray(x, dtype=np.float64)
        e = orc.knn_edges(x, knn, measure.sigma)
        rp, col, vals = orc.csr_from_edges(x.shape[0], e, orc.edge_weights(x, e, measure.sigma))
        return HostCsr(x.shape[0], x.shape[0], _t(rp, torch.int64), _t(col, torch.int64), _t(vals))

    def points(self, x):
        return np.ascontiguousarray(np.asarray(x, dtype=np.float64))

    def knn_select(self, x, knn, measure, p0, p1):
        # identity scan order; rows ascending like the device selection
        inv = -1.0 / measure.two_sigma_sq()
        sel = np.array([np.sort(orc.knn_select_row(x, i, knn, inv)) for i in range(p0, p1)],
                       dtype=np.int64).reshape(p1 - p0, knn)
        return _t(sel, torch.int32), _t(np.arange(x.shape[0]), torch.int32)

    def knn_union(self, x, knn, measure, sel, perm, r0, r1):
        sel, perm = sel.numpy().astype(np.int64), perm.numpy().astype(np.int64)
        n = x.shape[0]
        owner = np.repeat(perm, knn)  # point of each selection entry
        tgt = sel.ravel()
        # forward entries of local rows + reverse entries pointing into them
        fwd = (owner >= r0) & (owner < r1)
        rev = (tgt >= r0) & (tgt < r1)
        rows = np.concatenate((owner[fwd], tgt[rev]))
        cols = np.concatenate((tgt[fwd], owner[rev]))
        key = np.unique(rows * n + cols)
        rows, cols = key // n, key % n
        rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        np.add.at(rp, rows - r0 + 1, 1)
        lo, hi = np.minimum(rows, cols), np.maximum(rows, cols)  # once per unordered pair, i < j
        diff = x[lo] - x[hi]
        vals = np.exp(-np.einsum("ij,ij->i", diff, diff) / measure.two_sigma_sq())
        return HostCsr(r1 - r0, n, _t(np.cumsum(rp), torch.int64), _t(cols, torch.int64), _t(vals))

    def from_host_csr(self, m):
        return HostCsr(m.n_rows, m.n_cols, _t(m.row_ptr, torch.int64), _t(m.col_idx, torch.int64), _t(m.vals))

    def is_symmetric(self, w):
        a = np.zeros((w.n_rows, w.n_cols))
        rows = np.repeat(np.arange(w.n_rows), np.diff(w.row_ptr.numpy()))
        a[rows, w.col.numpy()] = w.vals.numpy()
        return w.n_rows == w.n_cols and np.array_equal(a, a.T)

    def slice_rows(self, w, r0, r1):
        rp = w.row_ptr[r0 : r1 + 1]
        b, e = int(rp[0]), int(rp[-1])
        return HostCsr(r1 - r0, w.n_cols, (rp - b).clone(), w.col[b:e].clone(), w.vals[b:e].clone())

    def degrees(self, a):
        return _t(orc.spmv_seq(a.row_ptr.numpy(), a.col.numpy(), a.vals.numpy(), np.ones(a.n_cols)))

    def zeros_count(self, d):
        return int((d == 0).sum())

    def sym_scale_shard(self, a, r0, d_full):
        rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr.numpy())) + r0
        d = d_full.numpy()
        return a.with_vals(_t(a.vals.numpy() / np.sqrt(d[rows] * d[a.col.numpy()])))

    # ---- Lanczos blocks (basis rows are vectors)
    def spmv(self, a, x_full):
        return _t(orc.spmv_seq(a.row_ptr.numpy(), a.col.numpy(), a.vals.numpy(), x_full.numpy()))

    def gemv_t(self, B, ncols, w):
        return _t(B[:ncols, : w.numel()].numpy() @ w.numpy())

    def gemv_n(self, B, ncols, h, w, want_sq=False):
        if ncols > 0:
            w -= _t(B[:ncols, : w.numel()].numpy().T @ h.numpy())
        if want_sq:
            return _t(np.array([float(w.numpy() @ w.numpy())]))
        return None

    def div_into(self, dst, src, div):
        dst.copy_(src / div)

    def normal(self, n, offset, seed, stream_id):
        # shard-independent: element g of the global vector depends on (seed, stream, g)
        full = np.random.default_rng([seed, stream_id]).standard_normal(offset + n)
        return _t(full[offset:])

    def symeig(self, T, k, p=None):
        theta, s = np.linalg.eigh(T)
        order = np.argsort(-theta, kind="stable")
        return theta[order], _t(s[:, order[:k]].T)

    def ritz(self, B, nl, m, S, k, rowmajor=False):
        y = S.numpy() @ B[:m, :nl].numpy()  # (k, nl)
        if rowmajor:
            return _t(y.T)
        out = torch.zeros((k, B.shape[1]), dtype=torch.float64)
        out[:, :nl] = _t(y)
        return out

    # ---- embedding
    def embed_scale(self, U, d_local):
        V = U.numpy() / np.sqrt(d_local.numpy())[:, None]
        return _t(V), _t((V * V).sum(axis=0))

    def embed_finish(self, V, colsq, normalize_rows):
        nrm = np.sqrt(colsq.numpy())
        nrm[nrm == 0.0] = 1.0
        v = V.numpy() / nrm
        if normalize_rows:
            v = orc.normalize_rows(v)
        return _t(v)

    # ---- k-means blocks
    def kmeans_assign(self, V, C, old):
        s = orc.pairwise_sq_dist(V.numpy(), C.numpy())
        lab = np.argmin(s, axis=1)
        cost = s[np.arange(len(lab)), lab]
        chg = 0 if old is None else int(np.count_nonzero(lab != old.numpy()))
        return _t(lab, torch.int64), _t(cost), chg, float(cost.sum())

    def local_sums(self, V, labels, k):
        v, lab = V.numpy(), labels.numpy()
        sums = np.zeros((k, v.shape[1]))
        np.add.at(sums, lab, v)
        return _t(sums), _t(np.bincount(lab, minlength=k), torch.int64)

    def divide(self, sums, counts):
        c = counts.numpy()
        out = np.zeros_like(sums.numpy())
        ne = c > 0
        out[ne] = sums.numpy()[ne] / c[ne, None]
        return _t(out)

    def farthest(self, cost_full, e):
        return np.argsort(-cost_full.numpy(), kind="stable")[:e]

    def kpp_session(self, V):
        return _NpKpp(V.numpy())

    def ncut_partials(self, a, r0, labels_full, k):
        lab = labels_full.numpy()
        rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr.numpy()))
        col, vals = a.col.numpy(), a.vals.numpy()
        li = lab[rows + r0]
        deg = np.bincount(rows, weights=vals, minlength=a.n_rows)
        cross = np.bincount(rows[li != lab[col]], weights=vals[li != lab[col]], minlength=a.n_rows)
        own = lab[r0 : r0 + a.n_rows]
        return (_t(np.bincount(own, weights=cross, minlength=k)), _t(np.bincount(own, weights=deg, minlength=k)),
                _t(np.bincount(own, minlength=k), torch.int64))


class _NpKpp:
    def __init__(self, v):
        self.v = v
        self.d2 = None
        self.taken = np.zeros(len(v), dtype=bool)
        self.total = 1.0

    def close(self):
        pass

    def take_row(self, row, local_index):
        diff = self.v - row.numpy()
        dist = np.einsum("ij,ij->i", diff, diff)
        self.d2 = dist if self.d2 is None else np.minimum(self.d2, dist)
        if local_index >= 0:
            self.taken[local_index] = True

    def _cand(self):
        return ~self.taken & (self.d2 > 0.0)

    def weight(self):
        c = self._cand()
        return float(self.d2[c].sum()), int(c.sum()), int((~self.taken).sum())

    def psum(self, total):
        self.total = total
        return float((self.d2[self._cand()] / total).sum())

    def search(self, target):
        idx = np.flatnonzero(self._cand())
        cum = np.cumsum(self.d2[idx] / self.total)
        hit = np.flatnonzero(cum > target)
        return int(idx[hit[0]]) if len(hit) else (int(idx[-1]) if len(idx) else -1)

    def nth_free(self, r):
        return int(np.flatnonzero(~self.taken)[r])
