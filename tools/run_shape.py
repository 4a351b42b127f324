"""One profiled end-to-end run of a blobs workload (bench.WORKLOADS name or
n,d,knn,k,cs) with stage times, eigen stats, kernel classes and quality."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import _native as nat  # noqa: E402
from paper_1802_04450_b200 import pipeline as pl  # noqa: E402

spec = sys.argv[1]
wl = bench.WORKLOADS[spec] if spec in bench.WORKLOADS else tuple(
    t(v) for t, v in zip((int, int, int, int, float), spec.split(",")))
n, d, knn, k, cs = wl
x, y = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
cfg = sc.PipelineConfig(
    input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))), pattern="knn", points=xd, knn=knn),
    k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
lib = nat.load()
lib.sc_profile_reset()
lib.sc_profile_enable(1)
torch.cuda.reset_peak_memory_stats()
t0 = time.perf_counter()
rep, w = pl.run_device(cfg)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
kc = {}
for c in ["knn_order", "knn_tile", "knn_recheck", "knn_fallback", "knn_union", "spmv", "reorth", "ritz", "symeig",
          "embed", "kmeanspp", "kmeans_assign", "kmeans_update", "ncut"]:
    ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
    lib.sc_profile_query(c.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
    if ms.value > 0:
        kc[c] = {"ms": round(ms.value, 2), "launches": cnt.value, "work": work.value}
out = {"workload": list(wl), "wall_s": wall, "stages_s": rep.timings, "nnz": w.nnz,
       "eigen": {a: b for a, b in pl.last_info.get("eigen", {}).items() if a != "history"},
       "kmeans_iters": rep.labeling.iters_run, "kernels": kc,
       "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
       "ari_vs_planted": float(sc.adjusted_rand_index(rep.labeling.labels, y)),
       "max_residual": float(np.max(rep.eigen_residuals)), "lambda": [float(rep.eigenvalues[0]),
                                                                     float(rep.eigenvalues[-1])],
       "warnings": rep.warnings}
print(json.dumps(out))
