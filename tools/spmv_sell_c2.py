"""Placed CSR SpMV vs the SELL-32-sigma operator on the C2 matrix in the
eigensolver's locality order: time per call, GB/s of the CSR algorithmic bytes,
and the SELL result's max deviation from the CSR one."""
import ctypes as C
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
st = nat.stream_handle()
xv = torch.randn(n, dtype=torch.float64, device="cuda")
y0 = torch.empty_like(xv)
y1 = torch.empty_like(xv)
nnz = a.nnz
by = nnz * 12 + (n + 1) * 8 + 2 * n * 8
rl = (a.row_ptr[1:] - a.row_ptr[:-1]).double()
out = {"n": n, "nnz": nnz, "alg_bytes": by, "row_len": [rl.min().item(), rl.mean().item(), rl.max().item()]}


def timeit(run, reps=100):
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def csr():
    nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv), nat.ptr(y0), 0, st))


h = C.c_void_p()
nat.check(lib.sc_sell_create(n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), st, C.byref(h)))
stored, nlong = C.c_int64(), C.c_int64()
lib.sc_sell_info(h, C.byref(stored), C.byref(nlong))
out["sell_stored"] = stored.value
out["sell_long_rows"] = nlong.value


def sell():
    nat.check(lib.sc_sell_spmv(h, nat.ptr(xv), nat.ptr(y1), st))


yseq = torch.empty_like(xv)
nat.check(lib.sc_spmv_f64(n, n, nat.ptr(a.row_ptr), nat.ptr(a.col), nat.ptr(a.vals), nat.ptr(xv), nat.ptr(yseq), 1, st))
for kind in sys.argv[2:] or ["placed"]:
    os.environ["SPECLUST_SPMV_KERNEL"] = kind
    t = timeit(csr)
    out[f"csr:{kind}"] = {"ms": t * 1e3, "GBs": by / t / 1e9, "max_dev_seq": (y0 - yseq).abs().max().item(),
                          "bit_exact_seq": bool(torch.equal(y0, yseq))}
for v in (os.environ.get("SPECLUST_SELL_VARIANTS") or "0").split(","):
    os.environ["SPECLUST_SELL_KERNEL"] = v
    t = timeit(sell)
    out[f"sell:{v}"] = {"ms": t * 1e3, "GBs": by / t / 1e9, "max_dev": (y1 - y0).abs().max().item()}
os.environ["SPECLUST_SPMV_KERNEL"] = "placed"
t = timeit(csr)
out["csr:placed:again"] = {"ms": t * 1e3, "GBs": by / t / 1e9}
lib.sc_sell_destroy(h)
print(json.dumps(out))
