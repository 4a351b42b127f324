"""Decomposition of the kNN candidate kernel at a blobs shape (profiling
switches of launch_tc2; every mode except 3 gives invalid lists):
3 = full kernel, 7 = MMA + TMA only, 19 = MMA + fast filter (no list code),
11 = epilogue without MMA, 27 = fast filter without MMA."""
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

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n, d, knn, k, cs = wl
x, _ = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
meas = sc.SimilarityMeasure.exp_decay(float(np.sqrt(d)))
lib = nat.load()
os.environ["SPECLUST_KNN_TILE_ONLY"] = "1"
out = {}
for mode in ["3", "7", "19", "11", "27", "3"]:
    os.environ["SPECLUST_KNN_WAIT"] = mode
    res = []
    for rep in range(2):
        lib.sc_profile_reset()
        lib.sc_profile_enable(1)
        try:
            knn_graph_device(xd, knn, meas)
        except Exception:
            pass
        torch.cuda.synchronize()
        lib.sc_profile_enable(0)
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(b"knn_tile", nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        res.append(round(ms.value, 2))
    out[mode] = res
print(json.dumps(out))
