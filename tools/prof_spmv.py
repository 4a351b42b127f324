"""Profile helper: build the C2 kNN graph, scale it (optionally permute it to
the kNN locality order), check the plan SpMV against the sequential kernel and
time both paths.  python tools/prof_spmv.py [perm|nat]"""
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
lab = rng.integers(0, k, n)
x = centers[lab] + rng.standard_normal((n, d))
w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(8.0))
a = sym_scale(w, degrees_device(w))
mode = sys.argv[1] if len(sys.argv) > 1 else "perm"
if mode == "perm":
    a, _ = permute_device(a, w.locality_perm)
elif mode == "ideal":  # points grouped by their true blob (upper bound on locality)
    a, _ = permute_device(a, torch.from_numpy(np.argsort(lab, kind="stable").astype(np.int32)).cuda())
lib = nat.load()
s = nat.stream_handle()
xv = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(xv)
yref = torch.empty_like(xv)
h = nat.C.c_void_p()
nat.check(lib.sc_spmv_plan_create(n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), s, nat.C.byref(h)))
nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv), nat.ptr(yref), 1, s))


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


nnz = a.nnz
alg = 12 * nnz + 8 * (n + 1) + 16 * n
for name, fn in [
    ("launch", lambda: nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals),
                                                 nat.ptr(xv), nat.ptr(y), 0, s))),
    ("plan", lambda: nat.check(lib.sc_spmv_plan_apply(h, nat.ptr(xv), nat.ptr(y), s))),
]:
    ms = timeit(fn)
    err = float(((y - yref).abs().max() / yref.abs().max()).item())
    print(f"{name:7s} mode={mode} nnz={nnz} spmv {ms:.4f} ms  {alg / ms / 1e6:.0f} GB/s  max rel err {err:.2e}")
lib.sc_spmv_plan_destroy(h)
