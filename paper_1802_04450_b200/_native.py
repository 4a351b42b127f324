"""ctypes binding of the C ABI declared in include/speclust_b200.h.

The shared library ``libspeclust_b200.so`` is built in-tree by
``__graft_entry__.build()``.  There is no CPU fallback: every compute entry
point of the package goes through this module, and a missing library or a
missing CUDA device raises ``NativeUnavailable`` at the first call.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

from . import errors

_LIB_PATH = Path(__file__).resolve().parent / "libspeclust_b200.so"
_lib = None

i64, i32, f64, vp = C.c_int64, C.c_int, C.c_double, C.c_void_p
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)
P_int = C.POINTER(C.c_int)


class LanczosStats(C.Structure):
    _fields_ = [
        ("restarts", C.c_int64),
        ("breakdowns", C.c_int64),
        ("matvecs", C.c_int64),
        ("n_history", C.c_int64),
        ("history", C.c_double * 512),
        ("second_passes", C.c_int64),
        ("flushes", C.c_int64),
        ("max_loss", C.c_double),
        ("mean_window", C.c_double),
    ]


# name -> (restype, argtypes); mirrors include/speclust_b200.h one-to-one
SIGNATURES = {
    "sc_last_error": (C.c_char_p, []),
    "sc_version": (i32, []),
    "sc_launch_count": (i64, []),
    "sc_launch_count_reset": (None, []),
    "sc_profile_enable": (None, [i32]),
    "sc_profile_reset": (None, []),
    "sc_profile_query": (i32, [C.c_char_p, P_f64, P_i64, P_f64]),
    "sc_spmv_f64": (i32, [i64, i64, vp, vp, vp, vp, vp, i32, vp]),
    "sc_degrees_f64": (i32, [i64, vp, vp, vp, vp]),
    "sc_find_nonpositive": (i32, [i64, vp, i32, P_i64, vp, i64, vp]),
    "sc_sym_scale_f64": (i32, [i64, vp, vp, vp, vp, vp, vp]),
    "sc_csr_is_symmetric": (i32, [i64, i64, vp, vp, vp, P_int, vp]),
    "sc_csr_validate": (i32, [i64, i64, i64, vp, vp, vp, vp]),
    "sc_trim_pool": (None, []),
    "sc_csr_permute_f64": (i32, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "sc_invert_perm": (i32, [i64, vp, vp, vp]),
    "sc_sell_create": (i32, [i64, vp, vp, vp, vp, C.POINTER(vp)]),
    "sc_sell_spmv": (i32, [vp, vp, vp, vp]),
    "sc_sell_info": (i32, [vp, P_i64, P_i64]),
    "sc_sell_destroy": (None, [vp]),
    "sc_spmv_plan_create": (i32, [i64, vp, vp, vp, vp, C.POINTER(vp)]),
    "sc_spmv_plan_apply": (i32, [vp, vp, vp, vp]),
    "sc_spmv_plan_destroy": (None, [vp]),
    "sc_gather_rows_f64": (i32, [i64, i64, vp, vp, vp, vp]),
    "sc_knn_graph_f64": (i32, [i64, i64, vp, i64, f64, vp, vp, vp, P_i64, P_i64, vp]),
    "sc_knn_select_f64": (i32, [i64, i64, vp, i64, f64, i64, i64, vp, vp, P_i64, vp]),
    "sc_knn_union_f64": (i32, [i64, i64, vp, i64, f64, vp, vp, i64, i64, vp, vp, vp, i64, P_i64, vp]),
    "sc_knn_select_vals_f64": (i32, [i64, i64, vp, i64, f64, i64, i64, vp, vp, vp, P_i64, vp]),
    "sc_knn_union_vals_f64": (i32, [i64, i64, vp, i64, f64, vp, vp, vp, i64, i64, vp, vp, vp, i64, P_i64, vp]),
    "sc_pair_weights": (i32, [i64, i64, vp, i64, vp, f64, vp, vp]),
    "sc_lanczos_create": (i32, [i64, i64, i64, f64, i64, C.c_uint64, vp, C.POINTER(vp)]),
    "sc_lanczos_destroy": (None, [vp]),
    "sc_lanczos_state": (i32, [vp]),
    "sc_lanczos_in_slot": (vp, [vp]),
    "sc_lanczos_out_slot": (vp, [vp]),
    "sc_lanczos_advance": (i32, [vp]),
    "sc_lanczos_get_stats": (i32, [vp, C.POINTER(LanczosStats)]),
    "sc_lanczos_ritz": (i32, [vp, P_f64, P_f64]),
    "sc_lanczos_extract": (i32, [vp, P_f64, vp]),
    "sc_eigensolve_csr": (i32, [i64, vp, vp, vp, i64, i64, f64, i64, C.c_uint64, P_f64, vp, P_f64,
                                C.POINTER(LanczosStats), vp]),
    "sc_eigensolve_csr_basis": (i32, [i64, vp, vp, vp, i64, i64, f64, i64, C.c_uint64, P_f64, vp, P_f64,
                                      C.POINTER(LanczosStats), vp]),
    "sc_lanczos_basis_ld": (i64, [i64]),
    "sc_eigensolve_csr_deflate": (i32, [i64, vp, vp, vp, vp, i64, i64, f64, i64, C.c_uint64, P_f64, vp, P_f64,
                                        C.POINTER(LanczosStats), C.POINTER(i64), vp]),
    "sc_recover_embedding_cm": (i32, [i64, i64, vp, i64, vp, i32, vp, vp]),
    "sc_symmetry_probe": (i32, [i64, vp, vp, vp, C.c_uint64, P_f64, vp]),
    "sc_recover_embedding": (i32, [i64, i64, vp, vp, i32, vp, vp]),
    "sc_normalize_rows": (i32, [i64, i64, vp, vp, vp]),
    "sc_pairwise_sq_dist": (i32, [i64, i64, i64, vp, vp, vp, vp]),
    "sc_kmeanspp_create": (i32, [i64, i64, vp, vp, C.POINTER(vp)]),
    "sc_kmeanspp_destroy": (None, [vp]),
    "sc_kmeanspp_take": (i32, [vp, i64]),
    "sc_kmeanspp_candidates": (i32, [vp, P_i64, P_i64]),
    "sc_kmeanspp_pick": (i32, [vp, i32, f64, i64, P_i64]),
    "sc_lloyd": (i32, [i64, i64, i64, vp, vp, i64, i64, vp, vp, P_f64, P_i64, vp]),
    "sc_ncut": (i32, [i64, vp, vp, vp, vp, i64, i32, P_f64, P_i64, vp]),
    "sc_partition_cuts": (i32, [i64, vp, vp, vp, vp, i64, P_f64, P_f64, P_i64, vp]),
    "sc_csr_remove_isolated": (i32, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, P_i64, P_i64, vp]),
    "sc_row_scale_f64": (i32, [i64, vp, vp, vp, vp, vp]),
    "sc_edge_similarity_f64": (i32, [i64, i64, vp, i64, vp, i32, i32, vp, P_i64, vp]),
    "sc_knn_graph_measure_f64": (i32, [i64, i64, vp, i64, i32, f64, i32, vp, vp, vp, P_i64, vp, P_i64, vp]),
    "sc_sbm_csr": (i32, [i64, vp, i64, f64, f64, C.c_uint64, vp, vp, vp, P_i64, vp]),
    "sc_pattern_edges_f64": (i32, [i64, i64, vp, i32, f64, f64, vp, P_i64, P_i64, vp]),
    "sc_gemv_t_f64": (i32, [i64, i64, i64, vp, vp, vp, vp]),
    "sc_gemv_n_f64": (i32, [i64, i64, i64, vp, vp, vp, vp, vp]),
    "sc_fill_normal": (i32, [i64, i64, C.c_uint64, C.c_uint64, vp, vp]),
    "sc_div_copy_f64": (i32, [i64, vp, f64, vp, vp]),
    "sc_symeig_f64": (i32, [i64, i64, vp, vp, vp, vp]),
    "sc_symeig_arrow_f64": (i32, [i64, i64, i64, vp, vp, vp, vp]),
    "sc_block_tn_f64": (i32, [i64, i64, i64, vp, vp, i64, vp, vp]),
    "sc_block_nn_f64": (i32, [i64, i64, i64, vp, vp, i64, vp, vp]),
    "sc_dgemm_tall": (i32, [i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, vp]),
    "sc_kmeans_assign": (i32, [i64, i64, i64, vp, vp, vp, vp, vp, P_i64, P_f64, vp]),
    "sc_kmeans_local_sums": (i32, [i64, i64, i64, vp, vp, vp, vp, vp]),
    "sc_centroid_divide": (i32, [i64, i64, vp, vp, vp, vp]),
    "sc_farthest": (i32, [i64, vp, i64, P_i64, vp]),
    "sc_kmeanspp_take_row": (i32, [vp, vp, i64]),
    "sc_kmeanspp_weight": (i32, [vp, P_f64, P_i64, P_i64]),
    "sc_kmeanspp_psum": (i32, [vp, f64, P_f64]),
    "sc_kmeanspp_search": (i32, [vp, f64, P_i64]),
    "sc_kmeanspp_nth_free": (i32, [vp, i64, P_i64]),
    "sc_sym_scale_shard_f64": (i32, [i64, i64, vp, vp, vp, vp, vp, vp]),
    "sc_embed_scale": (i32, [i64, i64, vp, vp, vp, vp, vp]),
    "sc_embed_finish": (i32, [i64, i64, vp, i32, vp, vp]),
    "sc_ncut_partials": (i32, [i64, i64, vp, vp, vp, vp, i64, vp, vp, vp, vp]),
}

# status code -> exception class (include/speclust_b200.h enum)
_STATUS = {
    -1: errors.BadConfig,
    -2: errors.DimensionMismatch,
    -3: errors.InvalidFormat,
    -4: errors.NotSquare,
    -5: errors.NotSymmetric,
    -6: errors.IsolatedNode,
    -7: errors.ZeroDegree,
    -8: errors.Breakdown,
    -9: errors.MaxRestartsExceeded,
    -10: errors.NotConverged,
    -11: errors.SpeclustError,
    -20: errors.NativeError,
    -21: errors.NativeError,
    -22: errors.NativeError,
}


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is no CPU path."""


def library_path() -> Path:
    return _LIB_PATH


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle with all signatures bound."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else _LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing: build it with `python __graft_entry__.py` (nvcc, sm_100a); "
            "this package has no CPU fallback"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    slow_ms = os.environ.get("SPECLUST_SLOW_MS")
    if slow_ms:  # diagnostics: report every library call slower than the threshold
        lib = _SlowLib(lib, float(slow_ms))
    if path is None:
        _lib = lib
    return lib


class _SlowLib:
    """SPECLUST_SLOW_MS=t: wraps the library so that every call taking more
    than t ms of host wall time is reported on stderr (with the time since
    the previous call returned, to tell a blocked call from host-side gaps)."""

    def __init__(self, lib, ms):
        import time

        self._lib, self._ms, self._time = lib, ms, time
        self._last = time.perf_counter()

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if not callable(fn) or name.startswith("_"):
            return fn
        t = self._time

        def wrapped(*a):
            t0 = t.perf_counter()
            gap = (t0 - self._last) * 1e3
            r = fn(*a)
            t1 = t.perf_counter()
            self._last = t1
            if (t1 - t0) * 1e3 > self._ms or gap > self._ms:
                sys.stderr.write(f"[slow] {name} {(t1 - t0) * 1e3:.1f} ms (gap before {gap:.1f} ms)\n")
            return r

        return wrapped


def last_error() -> str:
    msg = load().sc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, **payload):
    """Raise the errors.py class mapped from a status code."""
    if rc == 0:
        return
    cls = _STATUS.get(rc, errors.NativeError)
    msg = last_error()
    if cls is errors.IsolatedNode:
        raise cls(payload.get("indices", []))
    if cls is errors.MaxRestartsExceeded:
        raise cls(msg, values=payload.get("values"), residuals=payload.get("residuals"))
    raise cls(msg)


# ---------------------------------------------------------------------------
# torch handoff (device memory + streams only)
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the speclust_b200 engine runs on B200 only")
    return torch


def stream_handle():
    torch = torch_cuda()
    return vp(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> vp:
    return vp(t.data_ptr()) if t is not None else vp(0)


def empty_device(shape, dtype):
    """torch.empty on the device; on an out-of-memory error the library's
    cached pool is returned to the driver (sc_trim_pool) and PyTorch's own
    cache emptied once before retrying -- the multi-GB n x k tensors of the
    large configurations (C3: 32 GB each) land after stages whose buffers the
    library still caches."""
    torch = torch_cuda()
    try:
        return torch.empty(shape, dtype=dtype, device="cuda")
    except torch.OutOfMemoryError:
        load().sc_trim_pool()
        torch.cuda.empty_cache()
        return torch.empty(shape, dtype=dtype, device="cuda")


def to_device(a, dtype):
    """numpy / torch -> contiguous CUDA tensor of `dtype` (torch dtype)."""
    torch = torch_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:
        arr = arr.copy()
    return torch.from_numpy(arr).to(device="cuda", dtype=dtype, non_blocking=False).contiguous()


def to_host(t, dtype=None) -> np.ndarray:
    out = t.detach().cpu().numpy()
    if dtype is not None:
        out = out.astype(dtype, copy=False)
    return np.ascontiguousarray(out)


def frozen(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    a.flags.writeable = False
    return a
