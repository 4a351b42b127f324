"""One kNN graph build (blobs n, d, knn, k clusters, cs) on the device, for
ncu captures of the candidate kernel."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402

n, d, knn, k, cs = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5]))
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 1
x, _ = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
meas = sc.SimilarityMeasure.exp_decay(float(np.sqrt(d)))
for _ in range(reps):
    w = knn_graph_device(xd, knn, meas)
    torch.cuda.synchronize()
print("nnz", w.nnz)
