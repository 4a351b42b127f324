"""Sparse matrix types and operators (drop-in for speclust.sparse).

Host-facing types keep the reference contract (sparse.py:26-142): int64
indices, float64 values, read-only arrays, explicit zeros preserved, CSR
invariants validated on construction.  The compute operators (``spmv``,
``is_symmetric``) run on the GPU through the C ABI; ``DeviceCsr`` is the
device-resident form the pipeline keeps between stages:
``row_ptr`` int64[n+1], ``col`` int32[nnz], ``vals`` float64[nnz].
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import DimensionMismatch, DuplicateEntry, InvalidFormat

__all__ = [
    "CooMatrix",
    "CsrMatrix",
    "DeviceCsr",
    "coo_canonicalize",
    "coo_to_csr",
    "csr_to_coo",
    "spmv",
    "is_symmetric",
]


def _index_vec(a, what: str) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.int64)
    if out.ndim != 1:
        raise InvalidFormat(f"{what} must be one-dimensional")
    return out


def _value_vec(a) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.ndim != 1:
        raise InvalidFormat("vals must be one-dimensional")
    return out


def _check_dims(n_rows: int, n_cols: int):
    if n_rows < 0 or n_cols < 0:
        raise InvalidFormat("matrix dimensions must be nonnegative")


def _check_range(idx: np.ndarray, bound: int, what: str):
    if len(idx) and (idx.min() < 0 or idx.max() >= bound):
        raise InvalidFormat(f"{what} index out of range")


def _check_finite(vals: np.ndarray):
    if not np.isfinite(vals).all():
        raise InvalidFormat("matrix values must be finite")


@dataclass(frozen=True)
class CooMatrix:
    """(row, col, value) triplets; may be unsorted / duplicated until
    ``coo_canonicalize`` (reference sparse.py:46-80)."""

    n_rows: int
    n_cols: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    def __post_init__(self):
        rows, cols, vals = _index_vec(self.rows, "rows"), _index_vec(self.cols, "cols"), _value_vec(self.vals)
        _check_dims(self.n_rows, self.n_cols)
        if not (len(rows) == len(cols) == len(vals)):
            raise InvalidFormat("rows, cols, vals must have identical length")
        _check_range(rows, self.n_rows, "row")
        _check_range(cols, self.n_cols, "column")
        _check_finite(vals)
        for name, arr in (("rows", rows), ("cols", cols), ("vals", vals)):
            object.__setattr__(self, name, nat.frozen(arr))

    @property
    def nnz(self) -> int:
        return len(self.vals)


@dataclass(frozen=True)
class CsrMatrix:
    """Compressed sparse rows with strictly increasing columns per row
    (reference sparse.py:83-142)."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    _device: object = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "row_ptr", _index_vec(self.row_ptr, "row_ptr"))
        object.__setattr__(self, "col_idx", _index_vec(self.col_idx, "col_idx"))
        object.__setattr__(self, "vals", _value_vec(self.vals))
        self.validate()
        for name in ("row_ptr", "col_idx", "vals"):
            object.__setattr__(self, name, nat.frozen(getattr(self, name)))

    @property
    def nnz(self) -> int:
        return len(self.vals)

    def validate(self):
        """Raise InvalidFormat unless every CSR invariant holds."""
        _check_dims(self.n_rows, self.n_cols)
        rp, ci = self.row_ptr, self.col_idx
        if len(rp) != self.n_rows + 1:
            raise InvalidFormat("row_ptr must have length n_rows + 1")
        if len(ci) != len(self.vals):
            raise InvalidFormat("col_idx and vals must have identical length")
        if self.n_rows == 0:
            if self.nnz or rp[0] != 0:
                raise InvalidFormat("empty matrix must have empty row_ptr content")
            return
        if rp[0] != 0 or rp[-1] != self.nnz:
            raise InvalidFormat("row_ptr must start at 0 and end at nnz")
        if (np.diff(rp) < 0).any():
            raise InvalidFormat("row_ptr must be non-decreasing")
        if self.nnz:
            _check_range(ci, self.n_cols, "column")
            # within a row columns strictly increase; a step may only drop at a row start
            step_ok = np.diff(ci) > 0
            row_start = np.zeros(self.nnz - 1, dtype=bool)
            inner = rp[1:-1]
            inner = inner[(inner > 0) & (inner < self.nnz)]
            row_start[inner - 1] = True
            if not (step_ok | row_start).all():
                raise InvalidFormat("column indices must strictly increase within rows")
        _check_finite(self.vals)

    def row_indices(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_ptr))

    def device(self) -> "DeviceCsr":
        """Device copy (uploaded once, cached on the immutable matrix)."""
        if self._device is None:
            object.__setattr__(self, "_device", DeviceCsr.from_host(self))
        return self._device


class DeviceCsr:
    """Device-resident CSR (row_ptr int64, col int32, vals float64)."""

    def __init__(self, n_rows: int, n_cols: int, row_ptr, col, vals):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr, self.col, self.vals = row_ptr, col, vals

    @property
    def nnz(self) -> int:
        return int(self.col.numel())

    @classmethod
    def from_host(cls, m: CsrMatrix) -> "DeviceCsr":
        torch = nat.torch_cuda()
        if m.n_cols >= 2**31:
            raise InvalidFormat("device CSR needs n_cols < 2^31 (int32 columns)")
        return cls(m.n_rows, m.n_cols, nat.to_device(m.row_ptr, torch.int64),
                   nat.to_device(m.col_idx, torch.int32), nat.to_device(m.vals, torch.float64))

    def with_vals(self, vals) -> "DeviceCsr":
        return DeviceCsr(self.n_rows, self.n_cols, self.row_ptr, self.col, vals)

    def to_host(self) -> CsrMatrix:
        return CsrMatrix(self.n_rows, self.n_cols, nat.to_host(self.row_ptr),
                         nat.to_host(self.col, np.int64), nat.to_host(self.vals))


def coo_canonicalize(m: CooMatrix, dup_policy: str = "sum") -> CooMatrix:
    """Sort by (row, col) and merge duplicates (reference sparse.py:145-170).
    Host format conversion: it is not on the point-input hot path."""
    if dup_policy not in ("sum", "error"):
        raise ValueError(f"unknown dup_policy {dup_policy!r}")
    perm = np.lexsort((m.cols, m.rows))
    r, c, v = m.rows[perm], m.cols[perm], m.vals[perm]
    if len(r) > 1:
        same = (r[1:] == r[:-1]) & (c[1:] == c[:-1])
        if same.any():
            if dup_policy == "error":
                k = int(np.argmax(same))
                raise DuplicateEntry(f"duplicate entry at ({r[k]}, {c[k]})")
            first = np.flatnonzero(np.concatenate(([True], ~same)))
            r, c, v = r[first], c[first], np.add.reduceat(v, first)
    return CooMatrix(m.n_rows, m.n_cols, r, c, v)


def _is_canonical(m: CooMatrix) -> bool:
    if m.nnz < 2:
        return True
    r, c = m.rows, m.cols
    return bool(((r[1:] > r[:-1]) | ((r[1:] == r[:-1]) & (c[1:] > c[:-1]))).all())


def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """Row compression of a canonical COO (reference sparse.py:182-187)."""
    if not _is_canonical(m):
        raise InvalidFormat("COO matrix is not canonical; call coo_canonicalize")
    counts = np.bincount(m.rows, minlength=m.n_rows)
    row_ptr = np.zeros(m.n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CsrMatrix(m.n_rows, m.n_cols, row_ptr, m.cols, m.vals)


def csr_to_coo(m: CsrMatrix) -> CooMatrix:
    return CooMatrix(m.n_rows, m.n_cols, m.row_indices(), m.col_idx, m.vals)


def _as_device_csr(a) -> DeviceCsr:
    return a if isinstance(a, DeviceCsr) else a.device()


def spmv(a, x):
    """y = A x on the GPU, each row summed sequentially in column order —
    bit-identical to the reference (sparse.py:195-207).  Accepts a CsrMatrix
    (returns numpy) or a DeviceCsr with a CUDA tensor (returns a tensor)."""
    torch = nat.torch_cuda()
    dev_in = isinstance(x, torch.Tensor)
    xs = x if dev_in else np.asarray(x, dtype=np.float64)
    if tuple(xs.shape) != (a.n_cols,):
        raise DimensionMismatch(f"operand length {tuple(xs.shape)} does not match n_cols {a.n_cols}")
    d = _as_device_csr(a)
    xd = nat.to_device(xs, torch.float64)
    y = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    lib = nat.load()
    nat.check(lib.sc_spmv_f64(d.n_rows, d.n_cols, nat.ptr(d.row_ptr), nat.ptr(d.col), nat.ptr(d.vals),
                              nat.ptr(xd), nat.ptr(y), 1, nat.stream_handle()))
    return y if dev_in else nat.to_host(y)


def is_symmetric(a) -> bool:
    """Exact A == A^T check on the GPU (reference sparse.py:210-222)."""
    if a.n_rows != a.n_cols:
        return False
    if a.n_rows == 0:
        return True
    d = _as_device_csr(a)
    res = nat.C.c_int(0)
    lib = nat.load()
    nat.check(lib.sc_csr_is_symmetric(d.n_rows, d.nnz, nat.ptr(d.row_ptr), nat.ptr(d.col), nat.ptr(d.vals),
                                      nat.C.byref(res), nat.stream_handle()))
    return bool(res.value)
