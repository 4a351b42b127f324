"""One Lloyd call at the C5 shape (n rows, argv[1]) with max_iters argv[2] (ncu target)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200.kmeans import lloyd_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
it = int(sys.argv[2]) if len(sys.argv) > 2 else 1
v, init, lab = bench.make_c5(torch, n)
lloyd_device(v, init, sc.KmeansConfig(k=10_000, max_iters=it, init="random_points"))
torch.cuda.synchronize()
