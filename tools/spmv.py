import sys, time, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import _native as nat
from paper_1802_04450_b200.graph import knn_graph_device
from bench import make_blobs
x, _ = make_blobs(1_000_000, 64, 100, 0.7)
w = knn_graph_device(torch.from_numpy(x).cuda(), 32, sc.SimilarityMeasure.exp_decay(8.0))
n = w.n_rows
xv = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(xv)
lib = nat.load()
def run():
    nat.check(lib.sc_spmv_f64(n, n, nat.ptr(w.row_ptr), nat.ptr(w.col), nat.ptr(w.vals), nat.ptr(xv), nat.ptr(y), 0, nat.stream_handle()))
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
b = w.nnz * 12 + (n + 1) * 8 + 2 * n * 8
print(f"G={sys.argv[1] if len(sys.argv)>1 else 'auto'} nnz={w.nnz} {ms*1e3:.1f} us  {b/ms/1e6:.0f} GB/s")
