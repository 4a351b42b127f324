"""Locality statistics of the (optionally permuted) C2 operator + SpMV timing,
for ncu captures: python tools/spmv_locality.py [nat|perm]"""
import sys
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
y = rng.integers(0, k, n)
x = centers[y] + rng.standard_normal((n, d))
w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(8.0))
a = sym_scale(w, degrees_device(w))
mode = sys.argv[1] if len(sys.argv) > 1 else "perm"
if mode == "perm":
    a, _ = permute_device(a, w.locality_perm)
    perm = w.locality_perm.cpu().numpy()
    yb = y[perm]
else:
    yb = y
rp = a.row_ptr.cpu().numpy()
col = a.col.cpu().numpy().astype(np.int64)
rows = np.repeat(np.arange(n), np.diff(rp))
dist = np.abs(col - rows)
print(f"mode={mode} nnz={a.nnz} |col-row| quantiles 50/90/99: {np.percentile(dist, [50, 90, 99])}")
print(f"  same-blob neighbours: {np.mean(yb[rows] == yb[col]):.3f}")
print(f"  blob runs in the order: {1 + np.count_nonzero(yb[1:] != yb[:-1])}")
r = n // 148
for s in (0, 70):
    lo, hi = rp[s * r], rp[(s + 1) * r]
    lines = np.unique(col[lo:hi] // 16)
    print(f"  SM range {s}: {hi - lo} nnz touch {lines.size} x lines ({lines.size * 128 / 1024:.0f} KB)")
lib = nat.load()
xv = torch.randn(n, dtype=torch.float64, device="cuda")
yv = torch.empty_like(xv)
for _ in range(5):
    nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv), nat.ptr(yv), 0,
                              nat.stream_handle()))
torch.cuda.synchronize()
# windowed-SpMV hit fraction (spmv_window_kernel geometry: 148 row ranges,
# window of 26624 x entries centred on the range)
G, WIN = 148, 26624
hits = 0
for b in range(G):
    r0, r1 = n * b // G, n * (b + 1) // G
    half = max(0, (WIN - (r1 - r0)) // 2)
    wb = max(0, r0 - half)
    we = min(n, min(wb + WIN, r1 + half))
    c = col[rp[r0]:rp[r1]]
    hits += np.count_nonzero((c >= wb) & (c < we))
print(f"  window hit fraction {hits / col.size:.3f}")
