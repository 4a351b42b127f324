"""The CUDA per-shard path (CudaOps + Comm) at world sizes 2 and 3 on ONE
GPU: every rank is its own process on cuda:0, the collectives run over gloo
on the CUDA tensors (NCCL refuses two ranks on one device).  The sharded
pipeline (query-tile kNN graph + all-gather, row-block Lanczos, point-shard
k-means++ / Lloyd, sharded ncut) must give the same clustering as world 1
and the reference oracle."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import speclust_oracle as orc

pytestmark = pytest.mark.gpu

N, D, K, CS, KNN = 6000, 8, 6, 3.0, 12


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(sc, x):
    return sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(D))), pattern="knn", points=x,
                             knn=KNN),
        k_clusters=K, eigen=sc.LanczosConfig(k=K, seed=0), kmeans=sc.KmeansConfig(k=K, seed=0), normalize_rows=True)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1802_04450_b200 as sc
        from paper_1802_04450_b200 import distributed as dsc

        x, _ = orc.blobs(N, D, K, CS, seed=5)
        rep = dsc.run_sharded(_cfg(sc, x), dsc.Comm("cuda"), dsc.CudaOps())
        np.savez(os.path.join(out_dir, f"w{world}_r{rank}.npz"), labels=rep.labeling.labels,
                 values=rep.eigenvalues, residuals=rep.eigen_residuals, ncut=np.array(rep.ncut_value),
                 sse=rep.labeling.sse_history)
    finally:
        if world > 1:
            dist.destroy_process_group()


def _run(world, tmp_path):
    if world == 1:
        _worker(0, 1, 0, str(tmp_path))
    else:
        mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    out = []
    for r in range(world):
        with np.load(tmp_path / f"w{world}_r{r}.npz") as f:
            out.append({k: f[k] for k in f.files})
    return out


def test_cuda_shards_world_2_3_match_world_1_and_oracle(tmp_path):
    x, truth = orc.blobs(N, D, K, CS, seed=5)
    ref = orc.run_points(x, KNN, float(np.sqrt(D)), K)
    w1 = _run(1, tmp_path)[0]
    assert np.max(np.abs(w1["values"] - ref["values"]) / np.abs(ref["values"])) <= 1e-8
    assert orc.ari(w1["labels"], ref["labels"]) >= 0.999
    for world in (2, 3):
        res = _run(world, tmp_path)
        for r in res:  # replicated results are identical on every rank
            assert np.array_equal(r["labels"], res[0]["labels"])
            assert np.array_equal(r["values"], res[0]["values"])
        got = res[0]
        assert np.max(np.abs(got["values"] - w1["values"])) <= 1e-10
        assert orc.ari(got["labels"], w1["labels"]) == 1.0
        assert abs(float(got["ncut"]) - float(w1["ncut"])) <= 1e-10 * max(1.0, float(w1["ncut"]))
        assert np.all(got["residuals"] <= 1e-6)
    assert orc.ari(w1["labels"], truth) >= 0.99
