"""Profile helper: build the C2 kNN graph, scale it, and run the SpMV kernel
a few times (for ncu --kernel-name regex:spmv)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import _native as nat  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402
from paper_1802_04450_b200.laplacian import degrees_device, sym_scale  # noqa: E402
from paper_1802_04450_b200.pipeline import permute_device  # noqa: E402

n, d, knn, k, cs = 1_000_000, 64, 32, 100, 0.7
rng = np.random.default_rng(0)
centers = rng.normal(0.0, cs, (k, d))
x = centers[rng.integers(0, k, n)] + rng.standard_normal((n, d))
w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(8.0))
a = sym_scale(w, degrees_device(w))
mode = sys.argv[1] if len(sys.argv) > 1 else "perm"
if mode == "perm":
    a, _ = permute_device(a, w.locality_perm)
lib = nat.load()
xv = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(xv)
for _ in range(3):
    nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv), nat.ptr(y), 0,
                              nat.stream_handle()))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv), nat.ptr(y), 0,
                              nat.stream_handle()))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nnz = a.nnz
print(f"mode={mode} nnz={nnz} spmv {ms:.4f} ms  stream-bytes {(12 * nnz + 8 * n * 3 + 8 * n) / ms / 1e6:.0f} GB/s")
