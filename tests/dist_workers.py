"""Worker bodies for the multi-process (gloo, CPU) tests of the sharded
drivers; each returns a dict of numpy arrays saved by the test harness."""

from __future__ import annotations

import os

import numpy as np

import paper_1802_04450_b200 as sc
from oracle import speclust_oracle as orc
from paper_1802_04450_b200.distributed import Comm, lanczos_sharded, row_bounds, run_sharded
from paper_1802_04450_b200.errors import NotSymmetric
from tests.np_ops import HostCsr, NumpyOps


def random_symmetric(n=240, density=0.04, seed=3):
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    nz = int(density * n * n / 2)
    a[rng.integers(0, n, nz), rng.integers(0, n, nz)] = rng.standard_normal(nz)
    a = a + a.T
    r, c = np.nonzero(a)
    return a, sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, r, c, a[r, c])))


def lanczos_worker(rank, world):
    import torch

    _, m = random_symmetric()
    ops = NumpyOps()
    comm = Comm("cpu")
    n = m.n_rows
    bounds = row_bounds(n, comm.world)
    full = ops.from_host_csr(m)
    loc = ops.slice_rows(full, bounds[comm.rank], bounds[comm.rank + 1])
    vals, V, res, st = lanczos_sharded(ops, comm, loc, n, bounds, sc.LanczosConfig(k=6, seed=0))
    Vf = comm.gather_rows(V, bounds)
    return dict(values=vals, vectors=Vf.numpy(), residuals=res, restarts=st["restarts"], matvecs=st["matvecs"])


def blobs_cfg():
    x, truth = orc.blobs(360, 6, 4, 4.0, seed=11)
    cfg = sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(6.0))), pattern="knn", points=x,
                             knn=8),
        k_clusters=4, eigen=sc.LanczosConfig(k=4, seed=0), kmeans=sc.KmeansConfig(k=4, seed=0),
        normalize_rows=True)
    return x, truth, cfg


def pipeline_worker(rank, world):
    _, _, cfg = blobs_cfg()
    rep = run_sharded(cfg, Comm("cpu"), NumpyOps())
    return dict(labels=rep.labeling.labels, values=rep.eigenvalues, residuals=rep.eigen_residuals,
                ncut=np.array(rep.ncut_value), sse=rep.labeling.sse_history, centroids=rep.labeling.centroids)


def graph_worker(rank, world):
    from paper_1802_04450_b200.distributed import knn_graph_sharded

    x, _, cfg = blobs_cfg()
    comm = Comm("cpu")
    w, bounds = knn_graph_sharded(NumpyOps(), comm, x, 8, cfg.input.measure)
    nnz = comm.gather_scalars([w.nnz])[:, 0].astype(np.int64)
    rp = comm.gather_rows(w.row_ptr[1:], bounds)
    offs = np.concatenate(([0], np.cumsum(nnz)))
    rb = np.asarray(bounds)
    row_ptr = np.concatenate(([0], rp.numpy() + np.repeat(offs[:-1], np.diff(rb))))
    nb = [int(v) for v in offs]
    col = comm.gather_rows(w.col, nb).numpy()
    vals = comm.gather_rows(w.vals, nb).numpy()
    return dict(row_ptr=row_ptr, col=col, vals=vals)


def matrix_gates_worker(rank, world):
    """Sharded MatrixInput keeps the reference _resolve_graph gates
    (pipeline.py:181-192): NotSymmetric for A != A^T, a warning for negative
    weights."""
    a, m = random_symmetric(n=60, density=0.2, seed=5)
    a = np.abs(a) + np.eye(60)
    a[0, 1] += 0.5  # break symmetry in one entry
    r, c = np.nonzero(a)
    bad = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(60, 60, r, c, a[r, c])))
    cfg = sc.PipelineConfig(input=sc.MatrixInput(matrix=bad), k_clusters=2, eigen=sc.LanczosConfig(k=2, seed=0),
                            kmeans=sc.KmeansConfig(k=2, seed=0))
    raised = 0
    try:
        run_sharded(cfg, Comm("cpu"), NumpyOps())
    except NotSymmetric:
        raised = 1
    return dict(raised=np.array(raised))


def components_graph(nb=5, size=60, seed=9):
    """Block-diagonal nonnegative symmetric W: nb connected components."""
    rng = np.random.default_rng(seed)
    n = nb * size
    a = np.zeros((n, n))
    for b in range(nb):
        blk = rng.uniform(0.1, 1.0, (size, size)) * (rng.random((size, size)) < 0.3)
        blk = np.triu(blk, 1)
        blk = blk + blk.T
        # a path keeps every block connected
        for i in range(size - 1):
            blk[i, i + 1] = blk[i + 1, i] = max(blk[i, i + 1], 0.5)
        a[b * size:(b + 1) * size, b * size:(b + 1) * size] = blk
    r, c = np.nonzero(a)
    return a, sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, r, c, a[r, c])))


def deflate_worker(rank, world):
    """Row-sharded Lanczos on D^-1/2 W D^-1/2 of a 5-component graph with
    the eigenvalue-1 eigenvectors locked (distributed._LockedShards) and
    without (plain)."""
    os.environ["SPECLUST_DEFLATE_MIN_N"] = "100"
    _, m = components_graph()
    ops = NumpyOps()
    comm = Comm("cpu")
    n = m.n_rows
    bounds = row_bounds(n, comm.world)
    r0, r1 = bounds[comm.rank], bounds[comm.rank + 1]
    full = ops.from_host_csr(m)
    w_loc = ops.slice_rows(full, r0, r1)
    d_full = ops.degrees(full)
    a_loc = ops.sym_scale_shard(w_loc, r0, d_full)
    cfg = sc.LanczosConfig(k=8, seed=0)
    out = {}
    for tag, d in (("defl", d_full[r0:r1].contiguous()), ("plain", None)):
        vals, V, res, st = lanczos_sharded(ops, comm, a_loc, n, bounds, cfg, d_local=d)
        out[f"values_{tag}"] = vals
        out[f"residuals_{tag}"] = res
        out[f"vectors_{tag}"] = comm.gather_rows(V, bounds).numpy()
        out[f"locked_{tag}"] = np.array(st.get("locked", 0))
        out[f"restarts_{tag}"] = np.array(st["restarts"])
    return out


WORKERS = {"lanczos": lanczos_worker, "deflate": deflate_worker, "pipeline": pipeline_worker, "graph": graph_worker,
           "matrix_gates": matrix_gates_worker}


def spawn_entry(rank, world, port, name, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = WORKERS[name](rank, world)
        np.savez(os.path.join(out_dir, f"{name}_w{world}_r{rank}.npz"), **res)
    finally:
        if world > 1:
            dist.destroy_process_group()
