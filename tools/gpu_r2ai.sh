set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_shapes.py -q -x -k "knn or graph or pipeline or c3 or h3" > gpurun_out/ai_tests.log 2>&1
tail -3 gpurun_out/ai_tests.log
python - <<'PY' > gpurun_out/ai_modes.txt 2>&1
import os, sys, json, torch, numpy as np
sys.path.insert(0, ".")
import bench
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import _native as nat
from paper_1802_04450_b200.graph import knn_graph_device
lib = nat.load()
out = {}
for wl in ("c2", "c3h"):
    n, d, knn, k, cs = bench.WORKLOADS[wl]
    x, _ = bench.make_blobs(n, d, k, cs)
    xd = torch.from_numpy(x).cuda()
    for name, env in [("sorted", {}), ("nosort", {"SPECLUST_KNN_NOTILESORT": "1"}), ("sorted2", {})]:
        os.environ.pop("SPECLUST_KNN_NOTILESORT", None)
        os.environ.update(env)
        res = []
        for _ in range(2):
            lib.sc_profile_reset(); lib.sc_profile_enable(1)
            w = knn_graph_device(xd, knn, sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))))
            torch.cuda.synchronize(); lib.sc_profile_enable(0)
            ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
            lib.sc_profile_query(b"knn_tile", nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
            res.append(round(ms.value, 2))
        out[wl + "_" + name] = {"ms": res, "nnz": w.nnz}
    del xd
print(json.dumps(out))
PY
cat gpurun_out/ai_modes.txt
