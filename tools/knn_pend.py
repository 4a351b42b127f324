"""kNN candidate kernel time per list-append mode (SPECLUST_KNN_PEND)."""
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

n, d, knn, k, cs = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
x, _ = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
meas = sc.SimilarityMeasure.exp_decay(float(np.sqrt(d)))
lib = nat.load()
out = {}
for mode in sys.argv[2:] or ["0", "1,0", "2,0", "1,128", "2,128", "1,1024", "0"]:
    os.environ["SPECLUST_KNN_PEND"] = mode
    res = []
    for _ in range(2):
        lib.sc_profile_reset()
        lib.sc_profile_enable(1)
        w = knn_graph_device(xd, knn, meas)
        torch.cuda.synchronize()
        lib.sc_profile_enable(0)
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(b"knn_tile", nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        res.append(round(ms.value, 2))
    out[mode] = {"knn_tile_ms": res, "nnz": w.nnz}
print(json.dumps(out))
