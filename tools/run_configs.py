"""Scaled runs of BASELINE.json's larger configs on one GPU (shape checks and
timings, not bench lines):
  c3s: blobs N=120k, d=128, kNN=32, k=1000 (C3's large-k Lanczos, m=2000)
  c5s: k-means stress, 1M x 256 embedding, k=10,000, 20 Lloyd iterations
       from random_points init (C5's shape at 1/10 of the rows)
  c4g: C4's SBM graph at full size (16M nodes, 500 blocks, ~512M edges):
       device generation only
  c4s: C4 at 1/8 of the nodes (62 blocks x 32,000, same intra / inter
       degrees), MatrixInput -> eigensolve (k=62) -> k-means
python tools/run_configs.py [c3s] [c5s] [c4g] [c4s]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import _native as nat  # noqa: E402
from paper_1802_04450_b200.pipeline import last_info, run_device  # noqa: E402
from bench import make_blobs  # noqa: E402


def prof(lib, names):
    out = {}
    for nm in names:
        ms, c, w = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(nm.encode(), nat.C.byref(ms), nat.C.byref(c), nat.C.byref(w))
        if ms.value > 0:
            out[nm] = round(ms.value, 1)
    return out


lib = nat.load()
which = sys.argv[1:] or ["c3s", "c5s", "c4g", "c4s"]
if "c3s" in which:
    n, d, knn, k = 120_000, 128, 32, 1000
    x, y = make_blobs(n, d, k, 1.0)
    xd = torch.from_numpy(x).cuda()
    cfg = sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))), pattern="knn", points=xd,
                             knn=knn),
        k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep, w = run_device(cfg)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    ev = rep.eigenvalues
    print(f"c3s: {t:.2f} s stages {rep.timings} nnz {w.nnz} eigen {last_info.get('eigen')} "
          f"lambda[0] {ev[0]:.6f} lambda[k-1] {ev[-1]:.6f} "
          f"ARI vs blobs {sc.adjusted_rand_index(rep.labeling.labels, y):.4f} kernels {prof(lib, ['knn_tile', 'spmv', 'reorth', 'symeig', 'ritz', 'kmeans_assign', 'kmeanspp'])}",
          flush=True)
    lib.sc_profile_enable(0)
if "c5s" in which:
    n, d, k = 1_000_000, 256, 10_000
    rng = np.random.default_rng(0)
    centers = rng.standard_normal((k, d)).astype(np.float32)
    v = centers[rng.integers(0, k, n)] + 0.3 * rng.standard_normal((n, d)).astype(np.float32)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    vd = torch.from_numpy(v.astype(np.float64)).cuda()
    init = vd[torch.from_numpy(np.random.default_rng(0).choice(n, k, replace=False)).cuda()].contiguous()
    from paper_1802_04450_b200.kmeans import lloyd_device
    cfg = sc.KmeansConfig(k=k, max_iters=20, init="random_points")
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    labels, cent, hist, it = lloyd_device(vd, init, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"c5s: {t:.2f} s for {it} Lloyd iterations ({t / max(it, 1) * 1e3:.1f} ms/it) sse {hist[0]:.4e} -> "
          f"{hist[-1]:.4e} kernels {prof(lib, ['kmeans_assign', 'kmeans_update'])}", flush=True)
if "c4g" in which:
    from paper_1802_04450_b200.sbm import SbmConfig, sbm_generate_device
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    w, lab = sbm_generate_device(SbmConfig(block_sizes=(32_000,) * 500, p_in=1.6e-3, p_out=8.0e-7, seed=0))
    torch.cuda.synchronize()
    print(f"c4g: n={w.n_rows} nnz={w.nnz} ({w.nnz // 2} edges) generated in {time.perf_counter() - t0:.2f} s",
          flush=True)
    del w, lab
    torch.cuda.empty_cache()
if "c4s" in which:
    from paper_1802_04450_b200.sbm import SbmConfig, sbm_generate_device
    w, lab = sbm_generate_device(SbmConfig(block_sizes=(32_000,) * 62, p_in=1.6e-3, p_out=6.4e-6, seed=0))
    k = 62
    cfg = sc.PipelineConfig(input=sc.MatrixInput(matrix=w.to_host()), k_clusters=k,
                            eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0),
                            normalize_rows=True)
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep, _ = run_device(cfg)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"c4s: n={w.n_rows} nnz={w.nnz} {t:.2f} s stages {rep.timings} eigen {last_info.get('eigen')} "
          f"ARI vs blocks {sc.adjusted_rand_index(rep.labeling.labels, lab.cpu().numpy()):.4f} "
          f"kernels {prof(lib, ['spmv', 'reorth', 'symeig', 'ritz', 'kmeans_assign', 'kmeanspp'])}", flush=True)
