"""x footprint of the placed SpMV on the C2 operator (locality order): per
SM range (n/148 contiguous rows), the distinct x entries and distinct 32-byte
sectors its gathers touch, against the range's gather count."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import pipeline as pl  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402
from paper_1802_04450_b200.laplacian import degrees_device  # noqa: E402

n, d, knn, k, cs = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
x, _ = bench.make_blobs(n, d, k, cs)
w = knn_graph_device(torch.from_numpy(x).cuda(), knn, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
a = sc.sym_scale(w, degrees_device(w))
a, _ = pl.permute_device(a, w.locality_perm)
rp, col = a.row_ptr.long(), a.col.long()
out = {}
for nr in (148, 148 * 8):
    ent, sec, gat, span = [], [], [], []
    for i in range(nr):
        r0, r1 = n * i // nr, n * (i + 1) // nr
        c = col[rp[r0]:rp[r1]]
        ent.append(torch.unique(c).numel())
        sec.append(torch.unique(c // 4).numel())
        gat.append(c.numel())
        span.append((c.max() - c.min()).item())
    ent, sec, gat = np.array(ent), np.array(sec), np.array(gat)
    out[f"ranges_{nr}"] = {"rows_per_range": n // nr, "distinct_x_mean": float(ent.mean()), "distinct_x_max": int(ent.max()),
                           "distinct_sectors_mean": float(sec.mean()), "gathers_mean": float(gat.mean()),
                           "x_kb_mean": float(ent.mean() * 8 / 1024), "sector_kb_mean": float(sec.mean() * 32 / 1024),
                           "min_possible_l1_miss": float(sec.sum() / gat.sum()), "col_span_median": float(np.median(span))}
# fraction of nonzeros whose column lies within +-R rows
diff = (col - torch.repeat_interleave(torch.arange(n, device=col.device), (rp[1:] - rp[:-1]))).abs()
for R in (1024, 8192, 65536):
    out[f"frac_within_{R}"] = (diff <= R).double().mean().item()
print(json.dumps(out))
