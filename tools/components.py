"""Connected components of the kNN graphs of the bench workloads (min-label
propagation with pointer jumping in torch; a measurement tool)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402


def components(w):
    n = w.n_rows
    rows = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(w.row_ptr))
    cols = w.col.to(torch.int64)
    lab = torch.arange(n, device="cuda")
    for it in range(1000):
        m = lab.clone()
        m.scatter_reduce_(0, rows, lab[cols], reduce="amin")
        m = torch.minimum(m, m[m])  # pointer jumping
        if torch.equal(m, lab):
            break
        lab = m
    u, cnt = torch.unique(lab, return_counts=True)
    return int(u.numel()), it, cnt


out = {}
for wl in sys.argv[1:] or ["c2", "c3h", "c3"]:
    n, d, knn, k, cs = bench.WORKLOADS[wl]
    x, y = bench.make_blobs(n, d, k, cs)
    w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
    c, it, cnt = components(w)
    out[wl] = {"components": c, "iterations": it, "k": k, "largest": int(cnt.max()), "smallest": int(cnt.min())}
    del w
    torch.cuda.empty_cache()
print(json.dumps(out))
