"""kNN candidate kernel in chunked launches (SPECLUST_KNN_CHUNK CTAs per
launch): time of the knn_tile stage and CSR identity against one launch."""
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
meas = sc.SimilarityMeasure.exp_decay(float(np.sqrt(d)))
lib = nat.load()
ref = None
out = {}
for ch in sys.argv[2:]:
    os.environ["SPECLUST_KNN_CHUNK"] = ch
    knn_graph_device(xd, knn, meas)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        lib.sc_profile_reset()
        lib.sc_profile_enable(1)
        w = knn_graph_device(xd, knn, meas)
        torch.cuda.synchronize()
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(b"knn_tile", nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        times.append(round(ms.value, 2))
        lib.sc_profile_enable(0)
    col = w.col.cpu().numpy()
    if ref is None:
        ref = col
    out[ch] = {"knn_tile_ms": times, "same_csr": bool(np.array_equal(col, ref))}
print(json.dumps(out))
