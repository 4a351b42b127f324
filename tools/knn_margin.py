"""kNN candidate-kernel time and exact-fallback rows per candidate margin
(SPECLUST_KNN_MARGIN) at a bench workload; the CSR must not change."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import _native as nat  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, knn, k, cs = bench.WORKLOADS[wl]
x, _ = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
lib = nat.load()
out = {}
ref = None
for mg in sys.argv[2:] or ["24", "16", "12", "8"]:
    os.environ["SPECLUST_KNN_MARGIN"] = mg
    res = []
    for _ in range(2):
        lib.sc_profile_reset()
        lib.sc_profile_enable(1)
        torch.cuda.synchronize()
        import time
        t0 = time.perf_counter()
        w = knn_graph_device(xd, knn, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        lib.sc_profile_enable(0)
        q = {}
        for c in ("knn_tile", "knn_recheck", "knn_fallback", "knn_union"):
            ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
            lib.sc_profile_query(c.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
            q[c] = round(ms.value, 2)
        q["wall_ms"] = round(wall * 1e3, 1)
        res.append(q)
    if ref is None:
        ref = (w.row_ptr.clone(), w.col.clone(), w.vals.clone())
        same = True
    else:
        same = bool(torch.equal(ref[0], w.row_ptr) and torch.equal(ref[1], w.col) and torch.equal(ref[2], w.vals))
    out[mg] = {"runs": res, "csr_identical": same}
print(json.dumps(out))
