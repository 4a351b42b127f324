set -x
python - <<'PY' > gpurun_out/aa_modes.txt 2>&1
import os, sys, json, torch, numpy as np
sys.path.insert(0, ".")
import bench
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import _native as nat
from paper_1802_04450_b200.graph import knn_graph_device
n, d, knn, k, cs = bench.WORKLOADS["c2"]
x, _ = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
lib = nat.load()
os.environ["SPECLUST_KNN_TILE_ONLY"] = "1"
out = {}
for name, env in [("full", {}), ("nolist_compiled", {"SPECLUST_KNN_NOLIST": "1"}), ("mode19", {"SPECLUST_KNN_WAIT": "19"}), ("full2", {})]:
    for kk in ("SPECLUST_KNN_NOLIST", "SPECLUST_KNN_WAIT"):
        os.environ.pop(kk, None)
    os.environ.update(env)
    res = []
    for _ in range(2):
        lib.sc_profile_reset(); lib.sc_profile_enable(1)
        try:
            knn_graph_device(xd, knn, sc.SimilarityMeasure.exp_decay(8.0))
        except Exception:
            pass
        torch.cuda.synchronize(); lib.sc_profile_enable(0)
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(b"knn_tile", nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        res.append(round(ms.value, 2))
    out[name] = res
print(json.dumps(out))
PY
cat gpurun_out/aa_modes.txt
