"""Planted-partition stochastic block model (drop-in for speclust.sbm,
reference sbm.py:68-108), generated on the GPU straight into CSR.

Same configuration and validation as the reference (``SbmConfig``) and the
same distribution: every intra-block pair is an edge with probability
``p_in``, every inter-block pair with ``p_out``, independently.  The device
generator (``sc_sbm_csr``) flips each row's coins by geometric skipping over
a counter-based Philox stream, so its work is O(edges) and the C4 graph
(16M nodes, ~512M edges) is feasible; it is deterministic for a seed but does
not reproduce numpy's stream (parity is by distribution, see
tests/test_gpu_kernels.py::test_sbm_generator_statistics).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import BadConfig
from .sparse import CooMatrix, DeviceCsr, csr_to_coo

__all__ = ["SbmConfig", "sbm_generate", "sbm_generate_device"]


@dataclass(frozen=True)
class SbmConfig:
    block_sizes: tuple[int, ...]
    p_in: float
    p_out: float
    seed: int = 0

    def __post_init__(self):
        sizes = tuple(int(s) for s in self.block_sizes)
        object.__setattr__(self, "block_sizes", sizes)
        if len(sizes) == 0 or any(s < 1 for s in sizes):
            raise BadConfig("block_sizes must be a nonempty list of counts >= 1")
        if not 0.0 <= self.p_out <= self.p_in <= 1.0:
            raise BadConfig(f"need 0 <= p_out <= p_in <= 1, got p_in={self.p_in}, p_out={self.p_out}")


def sbm_generate_device(cfg: SbmConfig) -> tuple[DeviceCsr, object]:
    """One graph on the device: (symmetric unit-weight DeviceCsr without
    self-loops, int64 CUDA tensor of ground-truth block labels)."""
    torch = nat.torch_cuda()
    sizes = np.asarray(cfg.block_sizes, dtype=np.int64)
    offsets = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
    n = int(offsets[-1])
    od = nat.to_device(offsets, torch.int64)
    lib = nat.load()
    seed = int(cfg.seed) & (2**64 - 1)
    nnz = nat.C.c_int64()
    nat.check(lib.sc_sbm_csr(n, nat.ptr(od), len(sizes), float(cfg.p_in), float(cfg.p_out), seed, None, None, None,
                             nat.C.byref(nnz), nat.stream_handle()))
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(nnz.value, 1), dtype=torch.float64, device="cuda")
    nat.check(lib.sc_sbm_csr(n, nat.ptr(od), len(sizes), float(cfg.p_in), float(cfg.p_out), seed, nat.ptr(rp),
                             nat.ptr(col), nat.ptr(vals), nat.C.byref(nnz), nat.stream_handle()))
    labels = torch.repeat_interleave(torch.arange(len(sizes), device="cuda", dtype=torch.int64),
                                     torch.from_numpy(sizes).cuda())
    return DeviceCsr(n, n, rp, col[: nnz.value], vals[: nnz.value]), labels


def sbm_generate(cfg: SbmConfig) -> tuple[CooMatrix, np.ndarray]:
    """Draw one graph; returns (adjacency in canonical COO, ground-truth
    labels) like the reference's sbm_generate."""
    w, labels = sbm_generate_device(cfg)
    return csr_to_coo(w.to_host()), nat.to_host(labels)
