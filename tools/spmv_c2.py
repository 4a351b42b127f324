"""SpMV variants on the C2 operator in the eigensolver's locality order
(the matrix the Lanczos loop multiplies by): time per call and GB/s."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import _native as nat  # noqa: E402
from paper_1802_04450_b200 import pipeline as pl  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402
from paper_1802_04450_b200.laplacian import degrees_device  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n, d, knn, k, cs = wl
x, _ = bench.make_blobs(n, d, k, cs)
w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
deg = degrees_device(w)
a = sc.sym_scale(w, deg)
a, _ = pl.permute_device(a, w.locality_perm)
lib = nat.load()
xv = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(xv)
nnz = a.nnz
by = nnz * 12 + (n + 1) * 8 + 2 * n * 8
out = {"n": n, "nnz": nnz, "alg_bytes": by}
for i, kind in enumerate(["local", "placed", "pipe", "local", "placed"]):
    os.environ["SPECLUST_SPMV_KERNEL"] = kind
    st = nat.stream_handle()

    def run():
        nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv),
                                  nat.ptr(y), 0, st))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        run()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50 / 1e3
    out[f"{i}:{kind}"] = {"ms": t * 1e3, "GBs": by / t / 1e9}
print(json.dumps(out))
