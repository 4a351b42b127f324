"""Time the kNN candidate kernel alone (sc_profile knn_tile) at C2 shape."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import _native as nat
from paper_1802_04450_b200.graph import knn_graph_device
from bench import make_blobs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
x, _ = make_blobs(n, d, 100, 0.7)
xd = torch.from_numpy(x).cuda()
lib = nat.load()
try:
    knn_graph_device(xd, 32, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
except Exception as e:
    print("error", e)
torch.cuda.synchronize()
lib.sc_profile_reset(); lib.sc_profile_enable(1)
try:
    knn_graph_device(xd, 32, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
except Exception as e:
    print("error", e)
torch.cuda.synchronize()
out = []
for name in ["knn_order", "knn_tile", "knn_recheck", "knn_fallback", "knn_union"]:
    ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
    lib.sc_profile_query(name.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
    out.append(f"{name} {ms.value:.1f} ms")
    if name == "knn_tile" and ms.value > 0:
        out.append(f"({work.value / ms.value / 1e9:.0f} TFLOP/s)")
print(" ".join(out))
