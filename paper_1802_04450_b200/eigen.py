"""Restarted Lanczos eigensolver (drop-in for speclust.eigen).

Two entry styles, both backed by the device session ``sc_lanczos``:

* the reverse-communication interface of the paper / reference
  (``rci_new`` / ``rci_advance`` / ``rci_extract``, eigen.py:251-266): the
  caller applies the operator to ``in_slot`` and stores the product in
  ``out_slot``; the Krylov basis, reorthogonalisation, projected
  eigenproblem and thick restart all stay on the GPU;
* ``eigensolve`` (eigen.py:291-302), where the operator is a CSR matrix and
  the whole loop — SpMV included — runs on the device without returning to
  the host per matvec.

Semantics follow the reference: top-k algebraically largest pairs, subspace
size ``default_subspace_dim``, breakdown via fresh random directions, a
verification sweep before accepting a converged set, thick restart with an
arrowhead projection, true residuals in the result.  Random streams differ
from numpy's PCG64 (device Philox); results agree with the reference to
the Lanczos tolerance, not bit-for-bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import BadConfig, MaxRestartsExceeded, NotConverged, NotSquare, NotSymmetric, SpeclustError
from .sparse import CsrMatrix, DeviceCsr

__all__ = [
    "LanczosConfig",
    "EigenBasis",
    "RciSession",
    "default_subspace_dim",
    "rci_new",
    "rci_advance",
    "rci_extract",
    "eigensolve",
]

NEED_MATVEC = "need_matvec"
CONVERGED = "converged"
FAILED = "failed"
_STATES = {0: NEED_MATVEC, 1: CONVERGED, 2: FAILED}


def default_subspace_dim(n: int, k: int) -> int:
    """2k with a floor of k+8, capped at n (eigen.py:53-55)."""
    return min(n, max(2 * k, k + 8))


@dataclass(frozen=True)
class LanczosConfig:
    k: int
    m: int | None = None
    tol: float = 1e-8
    max_restarts: int = 300
    seed: int = 0


@dataclass(frozen=True)
class EigenBasis:
    """k pairs: values descending, unit-norm columns, true residuals."""

    values: np.ndarray
    vectors: np.ndarray
    residuals: np.ndarray

    def __post_init__(self):
        for name in ("values", "vectors", "residuals"):
            object.__setattr__(self, name, nat.frozen(np.asarray(getattr(self, name), dtype=np.float64)))


def _validate(n: int, cfg: LanczosConfig) -> int:
    m = cfg.m if cfg.m is not None else default_subspace_dim(n, cfg.k)
    if not (1 <= cfg.k < m <= n):
        raise BadConfig(f"need 1 <= k < m <= n, got k={cfg.k}, m={m}, n={n}")
    if not cfg.tol > 0:
        raise BadConfig(f"tol must be positive, got {cfg.tol}")
    if cfg.max_restarts < 0:
        raise BadConfig(f"max_restarts must be nonnegative, got {cfg.max_restarts}")
    return m


class _DevVec:
    """Zero-copy view of a library-owned device vector (CUDA array interface)."""

    def __init__(self, p: int, n: int, readonly: bool):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (p, False), "version": 3,
                                         "strides": None}


class RciSession:
    """Single-owner Lanczos state on the device (eigen.py:86-248).

    While ``state == "need_matvec"`` write ``A @ in_slot`` into ``out_slot``
    (numpy array or CUDA tensor of length n) and call ``rci_advance``.
    ``in_slot_device`` is a zero-copy CUDA view of the current vector.
    """

    def __init__(self, n: int, cfg: LanczosConfig):
        self.m = _validate(n, cfg)
        self.n, self.k, self.tol = n, cfg.k, float(cfg.tol)
        self.max_restarts = cfg.max_restarts
        self._lib = nat.load()
        handle = nat.vp()
        nat.check(self._lib.sc_lanczos_create(n, cfg.k, self.m, float(cfg.tol), cfg.max_restarts,
                                              int(cfg.seed) & (2**64 - 1), nat.stream_handle(), nat.C.byref(handle)))
        self._h = handle
        self.out_slot = np.zeros(n)
        self._refresh_in_slot()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.sc_lanczos_destroy(h)
            self._h = None

    # ---- reference-visible attributes
    @property
    def state(self) -> str:
        return _STATES[self._lib.sc_lanczos_state(self._h)]

    def _stats(self) -> nat.LanczosStats:
        st = nat.LanczosStats()
        self._lib.sc_lanczos_get_stats(self._h, nat.C.byref(st))
        return st

    @property
    def restart_count(self) -> int:
        return int(self._stats().restarts)

    @property
    def breakdown_count(self) -> int:
        return int(self._stats().breakdowns)

    @property
    def residual_history(self) -> list[float]:
        st = self._stats()
        return [float(st.history[i]) for i in range(st.n_history)]

    @property
    def in_slot_device(self):
        torch = nat.torch_cuda()
        p = self._lib.sc_lanczos_in_slot(self._h)
        return torch.as_tensor(_DevVec(p, self.n, True), device="cuda")

    def _refresh_in_slot(self):
        if self.state == NEED_MATVEC:
            self.in_slot = nat.frozen(nat.to_host(self.in_slot_device))

    def _ritz(self):
        vals = np.zeros(self.k)
        est = np.zeros(self.k)
        self._lib.sc_lanczos_ritz(self._h, vals.ctypes.data_as(nat.P_f64), est.ctypes.data_as(nat.P_f64))
        return vals, est

    def _advance(self) -> str:
        if self.state != NEED_MATVEC:
            raise SpeclustError(f"advance called in state {self.state!r}")
        torch = nat.torch_cuda()
        out = self.out_slot
        if isinstance(out, torch.Tensor):
            w = out.to(device="cuda", dtype=torch.float64).reshape(-1)
        else:
            w = np.asarray(out, dtype=np.float64)
            if w.shape != (self.n,):
                raise BadConfig(f"out_slot must have shape ({self.n},)")
            w = nat.to_device(w, torch.float64)
        if tuple(w.shape) != (self.n,):
            raise BadConfig(f"out_slot must have shape ({self.n},)")
        dst = torch.as_tensor(_DevVec(self._lib.sc_lanczos_out_slot(self._h), self.n, False), device="cuda")
        dst.copy_(w)
        rc = self._lib.sc_lanczos_advance(self._h)
        if rc == -9:
            vals, est = self._ritz()
            nat.check(rc, values=vals, residuals=est)
        nat.check(rc)
        self._refresh_in_slot()
        return self.state

    def _extract(self, apply) -> EigenBasis:
        if self.state != CONVERGED:
            raise NotConverged(f"extract called in state {self.state!r}")
        torch = nat.torch_cuda()
        vals = np.zeros(self.k)
        vecs = torch.empty((self.n, self.k), dtype=torch.float64, device="cuda")
        nat.check(self._lib.sc_lanczos_extract(self._h, vals.ctypes.data_as(nat.P_f64), nat.ptr(vecs)))
        v = nat.to_host(vecs)
        res = np.empty(self.k)
        for i in range(self.k):
            col = np.ascontiguousarray(v[:, i])
            res[i] = np.linalg.norm(np.asarray(apply(col), dtype=np.float64) - vals[i] * col)
        return EigenBasis(vals, v, res)


def rci_new(n: int, cfg: LanczosConfig) -> RciSession:
    return RciSession(n, cfg)


def rci_advance(session: RciSession) -> str:
    return session._advance()


def rci_extract(session: RciSession, apply) -> EigenBasis:
    return session._extract(apply)


def check_symmetric_device(a: DeviceCsr, seed: int):
    """Randomised symmetry probe (eigen.py:279-288) on the GPU."""
    ratio = nat.C.c_double(0.0)
    nat.check(nat.load().sc_symmetry_probe(a.n_rows, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals),
                                           (int(seed) * 2654435761 + 1) & (2**64 - 1), nat.C.byref(ratio),
                                           nat.stream_handle()))
    if ratio.value > 1e-10:
        raise NotSymmetric(f"asymmetry ratio {ratio.value:.3e} exceeds tolerance 1e-10")


def eigensolve_device(a: DeviceCsr, cfg: LanczosConfig, probe: bool = True):
    """Device-resident solve: returns (values numpy, vectors CUDA n x k,
    residuals numpy, stats dict)."""
    torch = nat.torch_cuda()
    if a.n_rows != a.n_cols:
        raise NotSquare(f"eigensolve requires a square matrix, got {a.n_rows}x{a.n_cols}")
    n = a.n_rows
    m = _validate(n, cfg)
    if probe:
        check_symmetric_device(a, cfg.seed)
    vals = np.zeros(cfg.k)
    res = np.zeros(cfg.k)
    vecs = nat.empty_device((n, cfg.k), torch.float64)
    st = nat.LanczosStats()
    rc = nat.load().sc_eigensolve_csr(n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), cfg.k, m,
                                      float(cfg.tol), cfg.max_restarts, int(cfg.seed) & (2**64 - 1),
                                      vals.ctypes.data_as(nat.P_f64), nat.ptr(vecs), res.ctypes.data_as(nat.P_f64),
                                      nat.C.byref(st), nat.stream_handle())
    if rc == -9:
        nat.check(rc, values=vals.copy(), residuals=res.copy())
    nat.check(rc)
    stats = dict(restarts=int(st.restarts), breakdowns=int(st.breakdowns), matvecs=int(st.matvecs),
                 second_passes=int(st.second_passes), flushes=int(st.flushes), max_loss=float(st.max_loss),
                 mean_window=float(st.mean_window),
                 history=[float(st.history[i]) for i in range(st.n_history)], m=m)
    return vals, vecs, res, stats


def eigensolve_device_deflate(a: DeviceCsr, d, cfg: LanczosConfig, probe: bool = True):
    """eigensolve_device for the normalized adjacency a = D^-1/2 W D^-1/2
    with its degrees d (CUDA, n): the eigenvalue-1 eigenvectors of the
    connected components are locked up front (sc_eigensolve_csr_deflate);
    stats["locked"] = their number (0: the plain solve ran)."""
    torch = nat.torch_cuda()
    if a.n_rows != a.n_cols:
        raise NotSquare(f"eigensolve requires a square matrix, got {a.n_rows}x{a.n_cols}")
    n = a.n_rows
    m = _validate(n, cfg)
    if probe:
        check_symmetric_device(a, cfg.seed)
    vals = np.zeros(cfg.k)
    res = np.zeros(cfg.k)
    vecs = nat.empty_device((n, cfg.k), torch.float64)
    st = nat.LanczosStats()
    locked = nat.C.c_int64(0)
    dd = d.to(device="cuda", dtype=torch.float64).contiguous()
    rc = nat.load().sc_eigensolve_csr_deflate(n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(dd),
                                              cfg.k, m, float(cfg.tol), cfg.max_restarts,
                                              int(cfg.seed) & (2**64 - 1), vals.ctypes.data_as(nat.P_f64),
                                              nat.ptr(vecs), res.ctypes.data_as(nat.P_f64), nat.C.byref(st),
                                              nat.C.byref(locked), nat.stream_handle())
    if rc == -9:
        nat.check(rc, values=vals.copy(), residuals=res.copy())
    nat.check(rc)
    stats = dict(restarts=int(st.restarts), breakdowns=int(st.breakdowns), matvecs=int(st.matvecs),
                 second_passes=int(st.second_passes), flushes=int(st.flushes), max_loss=float(st.max_loss),
                 mean_window=float(st.mean_window),
                 history=[float(st.history[i]) for i in range(st.n_history)], m=m, locked=int(locked.value))
    return vals, vecs, res, stats


def eigensolve_device_basis(a: DeviceCsr, cfg: LanczosConfig, probe: bool = True):
    """eigensolve_device with the Krylov basis as a caller-owned CUDA tensor
    ((m + 1) x ld, column j = basis vector j); the eigenvectors come back in
    its first k rows (column-major n x k with leading dimension ld) and no
    separate n x k result is allocated -- for operators where the basis and
    that result do not fit the device together (C4).  Returns (values,
    basis, ld, residuals, stats)."""
    torch = nat.torch_cuda()
    if a.n_rows != a.n_cols:
        raise NotSquare(f"eigensolve requires a square matrix, got {a.n_rows}x{a.n_cols}")
    n = a.n_rows
    m = _validate(n, cfg)
    if probe:
        check_symmetric_device(a, cfg.seed)
    lib = nat.load()
    ld = int(lib.sc_lanczos_basis_ld(n))
    basis = nat.empty_device((m + 1, ld), torch.float64)
    vals = np.zeros(cfg.k)
    res = np.zeros(cfg.k)
    st = nat.LanczosStats()
    rc = lib.sc_eigensolve_csr_basis(n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), cfg.k, m,
                                     float(cfg.tol), cfg.max_restarts, int(cfg.seed) & (2**64 - 1),
                                     vals.ctypes.data_as(nat.P_f64), nat.ptr(basis), res.ctypes.data_as(nat.P_f64),
                                     nat.C.byref(st), nat.stream_handle())
    if rc == -9:
        nat.check(rc, values=vals.copy(), residuals=res.copy())
    nat.check(rc)
    stats = dict(restarts=int(st.restarts), breakdowns=int(st.breakdowns), matvecs=int(st.matvecs),
                 second_passes=int(st.second_passes), flushes=int(st.flushes), max_loss=float(st.max_loss),
                 mean_window=float(st.mean_window),
                 history=[float(st.history[i]) for i in range(st.n_history)], m=m, in_basis=True)
    return vals, basis, ld, res, stats


def eigensolve(a, cfg: LanczosConfig) -> EigenBasis:
    """Top-k eigenpairs of a symmetric sparse matrix (eigen.py:291-302)."""
    if a.n_rows != a.n_cols:
        raise NotSquare(f"eigensolve requires a square matrix, got {a.n_rows}x{a.n_cols}")
    d = a if isinstance(a, DeviceCsr) else a.device()
    vals, vecs, res, _ = eigensolve_device(d, cfg)
    return EigenBasis(vals, nat.to_host(vecs), res)


_ = CsrMatrix  # re-exported type used in annotations by callers
_ = MaxRestartsExceeded
