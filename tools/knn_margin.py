"""kNN candidate margin sweep at C2: kernel time and rows needing the exact fallback."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import _native as nat  # noqa: E402
from paper_1802_04450_b200.graph import knn_graph_device  # noqa: E402
from bench import make_blobs  # noqa: E402

x, _ = make_blobs(1_000_000, 64, 100, 0.7)
xd = torch.from_numpy(x).cuda()
lib = nat.load()
m = sc.SimilarityMeasure.exp_decay(8.0)
knn_graph_device(xd, 32, m)
torch.cuda.synchronize()
lib.sc_profile_reset()
lib.sc_profile_enable(1)
w, st = knn_graph_device(xd, 32, m, return_stats=True)
torch.cuda.synchronize()
ms = {}
for name in ["knn_tile", "knn_recheck", "knn_fallback"]:
    t, c, wk = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
    lib.sc_profile_query(name.encode(), nat.C.byref(t), nat.C.byref(c), nat.C.byref(wk))
    ms[name] = round(t.value, 1)
print(os.environ.get("SPECLUST_KNN_MARGIN"), ms, st)
