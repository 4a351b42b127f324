"""How much of the C2 SpMV is the x gathers: the placed kernel on the real
locality-ordered operator vs the same matrix with every column index set to
its row (no gathers: a pure stream) and the |col - row| distribution."""
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

n, d, knn, k, cs = bench.WORKLOADS["c2"]
x, _ = bench.make_blobs(n, d, k, cs)
w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
deg = degrees_device(w)
a = sc.sym_scale(w, deg)
a, _ = pl.permute_device(a, w.locality_perm)
lib = nat.load()
xv = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(xv)
nnz = a.nnz
rows = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int64), torch.diff(a.row_ptr))
dist = (a.col.to(torch.int64) - rows).abs()
out = {"n": n, "nnz": nnz}
for W in (64, 256, 1024, 4096, 16384, 65536):
    out[f"frac_within_{W}"] = float((dist < W).float().mean())
by = nnz * 12 + (n + 1) * 8 + 2 * n * 8
st = nat.stream_handle()


def timeit(col):
    def run():
        nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(col), nat.ptr(a.vals), nat.ptr(xv),
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
    return {"ms": round(t * 1e3, 4), "GBs": round(by / t / 1e9, 1)}


col_self = rows.to(torch.int32)
col_shift = ((rows + 37) % n).to(torch.int32)
for kind in ("placed", "local"):
    os.environ["SPECLUST_SPMV_KERNEL"] = kind
    out[kind + "_real"] = timeit(a.col)
    out[kind + "_self"] = timeit(col_self)
    out[kind + "_shift37"] = timeit(col_shift)
# the bulk-staged plan kernels (cp.async.bulk ring, SpmvPlan)
import itertools  # noqa: E402
for kind, (name, col) in itertools.product(("bulk",), (("real", a.col), ("self", col_self))):
    os.environ["SPECLUST_SPMV_KERNEL"] = kind
    h = nat.vp()
    nat.check(lib.sc_spmv_plan_create(n, nat.ptr(a.row_ptr), nat.ptr(col), nat.ptr(a.vals), st, nat.C.byref(h)))

    def runp():
        nat.check(lib.sc_spmv_plan_apply(h, nat.ptr(xv), nat.ptr(y), st))
    runp()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        runp()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50 / 1e3
    if kind == "stream" and name == "real":
        ref = torch.empty_like(y)
        os.environ["SPECLUST_SPMV_KERNEL"] = "placed"
        nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv),
                                  nat.ptr(ref), 0, st))
        torch.cuda.synchronize()
        out["stream_vs_placed_maxrel"] = float(((y - ref).abs().max() / ref.abs().max()).item())
    out[kind + "_" + name] = {"ms": round(t * 1e3, 4), "GBs": round(by / t / 1e9, 1)}
    lib.sc_spmv_plan_destroy(h)
print(json.dumps(out))
