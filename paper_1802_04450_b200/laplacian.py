"""Degrees and normalised operators (drop-in for speclust.laplacian).

The pipeline takes the top-k eigenpairs of A = D^-1/2 W D^-1/2 and maps them
back to eigenvectors of D^-1 W (reference laplacian.py:1-9).  ``degrees``,
``sym_scale`` and ``recover_row_eigvecs`` run on the GPU; ``degrees`` and
``sym_scale`` reproduce the reference bit-for-bit (sequential row sums; one
IEEE product, square root and division per entry).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .errors import DimensionMismatch, IsolatedNode, NotSquare, ZeroDegree
from .sparse import CsrMatrix, DeviceCsr

__all__ = ["degrees", "handle_isolated", "row_scale", "sym_scale", "recover_row_eigvecs"]


def _dev(w):
    return w if isinstance(w, DeviceCsr) else w.device()


def degrees_device(w: DeviceCsr):
    torch = nat.torch_cuda()
    d = torch.empty(w.n_rows, dtype=torch.float64, device="cuda")
    nat.check(nat.load().sc_degrees_f64(w.n_rows, nat.ptr(w.row_ptr), nat.ptr(w.vals), nat.ptr(d),
                                        nat.stream_handle()))
    return d


def degrees(w) -> np.ndarray:
    """Row sums of W (reference laplacian.py:27-31)."""
    if w.n_rows != w.n_cols:
        raise NotSquare(f"degree computation requires a square matrix, got {w.n_rows}x{w.n_cols}")
    d = degrees_device(_dev(w))
    return d if isinstance(w, DeviceCsr) else nat.to_host(d)


def nonpositive_device(d, mode: int, max_list: int = 0):
    """(count, first indices) of d == 0 (mode 0) or d <= 0 (mode 1)."""
    torch = nat.torch_cuda()
    cnt = nat.C.c_int64(0)
    idx = torch.empty(max(1, max_list), dtype=torch.int64, device="cuda")
    nat.check(nat.load().sc_find_nonpositive(int(d.numel()), nat.ptr(d), mode, nat.C.byref(cnt), nat.ptr(idx),
                                             max_list, nat.stream_handle()))
    c = cnt.value
    return c, (nat.to_host(idx[: min(c, max_list)]) if c and max_list else np.zeros(0, dtype=np.int64))


def handle_isolated(w, d, policy: str = "error"):
    """Zero-degree handling before normalisation (reference
    laplacian.py:34-64): 'error' raises IsolatedNode(indices); 'remove'
    returns the induced submatrix, its degrees and the old->new remap."""
    if policy not in ("error", "remove"):
        raise ValueError(f"unknown isolated-node policy {policy!r}")
    torch = nat.torch_cuda()
    dev = isinstance(d, torch.Tensor)
    dd = d if dev else nat.to_device(np.asarray(d, dtype=np.float64), torch.float64)
    n = int(dd.numel())
    count, _ = nonpositive_device(dd, 0)
    identity = np.arange(n, dtype=np.int64)
    if count == 0:
        return w, d, identity
    _, idx = nonpositive_device(dd, 0, count)
    if policy == "error":
        raise IsolatedNode(idx)
    # 'remove' (input cleaning): induced submatrix on device
    dw = _dev(w)
    remap = torch.empty(n, dtype=torch.int64, device="cuda")
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty_like(dw.col)
    vals = torch.empty_like(dw.vals)
    d_out = torch.empty(n, dtype=torch.float64, device="cuda")
    n_new, nnz_new = nat.C.c_int64(), nat.C.c_int64()
    nat.check(nat.load().sc_csr_remove_isolated(n, nat.ptr(dw.row_ptr), nat.ptr(dw.col), nat.ptr(dw.vals),
                                                nat.ptr(dd), nat.ptr(remap), nat.ptr(rp), nat.ptr(col),
                                                nat.ptr(vals), nat.ptr(d_out), nat.C.byref(n_new),
                                                nat.C.byref(nnz_new), nat.stream_handle()))
    m, z = n_new.value, nnz_new.value
    sub = DeviceCsr(m, m, rp[: m + 1], col[:z], vals[:z])
    if isinstance(w, DeviceCsr):
        return sub, d_out[:m], nat.to_host(remap)
    return sub.to_host(), nat.to_host(d_out[:m]), nat.to_host(remap)


def _positive(d):
    torch = nat.torch_cuda()
    dd = d if isinstance(d, torch.Tensor) else nat.to_device(np.asarray(d, dtype=np.float64), torch.float64)
    count, idx = nonpositive_device(dd, 1, 1)
    if count:
        raise ZeroDegree(f"non-positive degree at node {int(idx[0])}")
    return dd


def sym_scale(w, d):
    """a_ij = w_ij / sqrt(d_i d_j) (reference laplacian.py:84-91)."""
    torch = nat.torch_cuda()
    dd = _positive(d)
    if int(dd.numel()) != w.n_rows:
        raise DimensionMismatch(f"degree vector length {int(dd.numel())} does not match n_rows {w.n_rows}")
    dw = _dev(w)
    out = torch.empty_like(dw.vals)
    nat.check(nat.load().sc_sym_scale_f64(dw.n_rows, nat.ptr(dw.row_ptr), nat.ptr(dw.col), nat.ptr(dw.vals),
                                          nat.ptr(dd), nat.ptr(out), nat.stream_handle()))
    res = dw.with_vals(out)
    if isinstance(w, DeviceCsr):
        return res
    return CsrMatrix(w.n_rows, w.n_cols, w.row_ptr, w.col_idx, nat.to_host(out))


def row_scale(w, d) -> CsrMatrix:
    """Row-stochastic D^-1 W (reference laplacian.py:75-81) on device:
    out = vals / d[row] with IEEE division (bit-identical)."""
    torch = nat.torch_cuda()
    dd = _positive(d)
    if int(dd.numel()) != w.n_rows:
        raise DimensionMismatch(f"degree vector length {int(dd.numel())} does not match n_rows {w.n_rows}")
    dw = _dev(w)
    out = torch.empty_like(dw.vals)
    nat.check(nat.load().sc_row_scale_f64(dw.n_rows, nat.ptr(dw.row_ptr), nat.ptr(dw.vals), nat.ptr(dd),
                                          nat.ptr(out), nat.stream_handle()))
    res = dw.with_vals(out)
    if isinstance(w, DeviceCsr):
        return res
    return CsrMatrix(w.n_rows, w.n_cols, w.row_ptr, w.col_idx, nat.to_host(out))


def recover_embedding_device(u, d, normalize_rows: bool):
    """v = u / sqrt(d) rowwise, unit columns, optionally unit rows; u is a
    CUDA (n, k) float64 tensor."""
    torch = nat.torch_cuda()
    n, k = u.shape
    out = nat.empty_device(tuple(u.shape), u.dtype)
    nat.check(nat.load().sc_recover_embedding(n, k, nat.ptr(u), nat.ptr(d), 1 if normalize_rows else 0,
                                              nat.ptr(out), nat.stream_handle()))
    return out


def recover_embedding_from_basis(basis, ld: int, n: int, k: int, d, normalize_rows: bool):
    """recover_embedding_device for eigenvectors left in the Lanczos basis
    (eigen.eigensolve_device_basis: rows 0..k-1 of `basis`, each a vector of
    length ld).  The row-major n x k embedding is written into the basis rows
    k..2k-1 when the basis has them (a view: no new n x k allocation), else
    into a new tensor."""
    torch = nat.torch_cuda()
    flat = basis.view(-1)
    if basis.shape[0] >= 2 * k:
        out = flat[k * ld: k * ld + n * k].view(n, k)
    else:
        out = nat.empty_device((n, k), torch.float64)
    nat.check(nat.load().sc_recover_embedding_cm(n, k, nat.ptr(basis), ld, nat.ptr(d), 1 if normalize_rows else 0,
                                                 nat.ptr(out), nat.stream_handle()))
    return out


def recover_row_eigvecs(u, d):
    """Eigenvectors of the symmetric form -> eigenvectors of D^-1 W with unit
    columns (reference laplacian.py:94-106)."""
    torch = nat.torch_cuda()
    dd = _positive(d)
    dev = isinstance(u, torch.Tensor)
    if not dev:
        u = np.asarray(u, dtype=np.float64)
    if u.ndim != 2 or u.shape[0] != int(dd.numel()):
        raise DimensionMismatch(f"eigenvector matrix shape {tuple(u.shape)} does not match degree length {int(dd.numel())}")
    if u.shape[1] == 0:
        return u.clone() if dev else u.copy()
    ud = nat.to_device(u, torch.float64)
    out = recover_embedding_device(ud, dd, False)
    return out if dev else nat.to_host(out)
