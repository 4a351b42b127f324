"""Profile helper: one C2 clustering through the public device pipeline (used
under ncu with a kernel filter, e.g. the Lanczos reorthogonalisation GEMVs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04450_b200 as sc  # noqa: E402
from bench import make_blobs  # noqa: E402
from paper_1802_04450_b200.pipeline import run_device  # noqa: E402

n, d, knn, k, cs = 1_000_000, 64, 32, 100, 0.7
x, _ = make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
sigma = float(np.sqrt(d))
cfg = sc.PipelineConfig(
    input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(sigma), pattern="knn", points=xd, knn=knn),
    k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
rep, _ = run_device(cfg)
torch.cuda.synchronize()
print("ok", rep.eigenvalues[:3])
