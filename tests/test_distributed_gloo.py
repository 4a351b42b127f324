"""Multi-process (gloo, CPU) coverage of the sharded drivers: row-sharded
Lanczos and the sharded pipeline (row-sharded eigen + point-sharded
k-means++/Lloyd + sharded ncut) at world sizes 1, 2 and 3 must agree with each
other and with the CPU oracle.  Per-shard compute is the numpy ops of
tests/np_ops.py; the collectives are the product code's (Comm)."""

import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import speclust_oracle as orc
from tests import dist_workers as dw


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(name, world, tmp_path):
    if world == 1:
        dw.spawn_entry(0, 1, 0, name, str(tmp_path))
    else:
        mp.spawn(dw.spawn_entry, args=(world, _port(), name, str(tmp_path)), nprocs=world, join=True)
    out = []
    for r in range(world):
        with np.load(tmp_path / f"{name}_w{world}_r{r}.npz") as f:
            out.append({k: f[k] for k in f.files})
    return out


def test_lanczos_sharded_matches_single_and_lapack(tmp_path):
    a, _ = dw.random_symmetric()
    want = np.sort(np.linalg.eigvalsh(a))[::-1][:6]
    w1 = run_world("lanczos", 1, tmp_path)[0]
    for world in (2, 3):
        res = run_world("lanczos", world, tmp_path)
        for r in res:  # every rank holds the same replicated result
            assert np.array_equal(r["values"], res[0]["values"])
        got = res[0]
        assert np.max(np.abs(got["values"] - want)) <= 1e-8
        assert np.max(np.abs(got["values"] - w1["values"])) <= 1e-10
        assert int(got["restarts"]) == int(w1["restarts"])
        assert np.all(got["residuals"] <= 1e-6)
        v = got["vectors"]
        assert np.abs(v.T @ v - np.eye(6)).max() <= 1e-8


def test_pipeline_sharded_matches_oracle(tmp_path):
    x, truth, _ = dw.blobs_cfg()
    ref = orc.run_points(x, 8, float(np.sqrt(6.0)), 4)
    w1 = run_world("pipeline", 1, tmp_path)[0]
    for world in (2, 3):
        res = run_world("pipeline", world, tmp_path)
        for r in res:
            assert np.array_equal(r["labels"], res[0]["labels"])
        got = res[0]
        assert np.max(np.abs(got["values"] - ref["values"]) / np.abs(ref["values"])) <= 1e-8
        assert orc.ari(got["labels"], ref["labels"]) >= 0.999
        assert orc.ari(got["labels"], w1["labels"]) == 1.0
        assert abs(float(got["ncut"]) - ref["ncut"]) <= 1e-10 * max(1.0, ref["ncut"])
        assert orc.ari(got["labels"], truth) >= 0.99


def test_knn_graph_sharded_rows_match_oracle(tmp_path):
    """Query-tile sharded selection + all-gather + per-rank union reassembles
    the reference CSR bit for bit (graph.py:185-237)."""
    x, _, _ = dw.blobs_cfg()
    e = orc.knn_edges(x, 8, float(np.sqrt(6.0)))
    rp, col, vals = orc.csr_from_edges(x.shape[0], e, orc.edge_weights(x, e, float(np.sqrt(6.0))))
    for world in (2, 3):
        got = run_world("graph", world, tmp_path)[0]
        assert np.array_equal(got["row_ptr"], rp)
        assert np.array_equal(got["col"], col)
        assert np.array_equal(got["vals"], vals)


def test_sharded_matrix_input_symmetry_gate(tmp_path):
    for world in (1, 2):
        for r in run_world("matrix_gates", world, tmp_path):
            assert int(r["raised"]) == 1


@pytest.mark.parametrize("world", [1, 2, 3])
def test_row_bounds_partition(world):
    from paper_1802_04450_b200.distributed import row_bounds

    b = row_bounds(10, world)
    assert b[0] == 0 and b[-1] == 10 and all(b[i] <= b[i + 1] for i in range(world))
    sizes = np.diff(b)
    assert sizes.max() - sizes.min() <= 1


def test_lanczos_sharded_locked_components(tmp_path):
    """Sharded counterpart of sc_eigensolve_csr_deflate: on a 5-component
    graph the eigenvalue-1 eigenvectors (one per component) are locked and the
    rest solved on their complement; eigenvalues, residuals and the
    eigenvalue-1 eigenspace agree with the plain sharded solve and LAPACK at
    world sizes 1, 2 and 3."""
    a, _ = dw.components_graph()
    d = a.sum(axis=1)
    s = a / np.sqrt(np.outer(d, d))
    want = np.sort(np.linalg.eigvalsh(s))[::-1][:8]
    for world in (1, 2, 3):
        res = run_world("deflate", world, tmp_path)
        got = res[0]
        for r in res:
            assert np.array_equal(r["values_defl"], got["values_defl"])
        assert int(got["locked_defl"]) == 5 and int(got["locked_plain"]) == 0
        assert np.max(np.abs(got["values_defl"] - want)) <= 1e-9
        assert np.max(np.abs(got["values_plain"] - want)) <= 1e-9
        assert np.max(np.abs(got["values_defl"][:5] - 1.0)) <= 1e-12
        assert np.all(got["residuals_defl"] <= 1e-7)
        v = got["vectors_defl"]
        assert np.abs(v.T @ v - np.eye(8)).max() <= 1e-9
        q1, _ = np.linalg.qr(v[:, :5])
        q2, _ = np.linalg.qr(got["vectors_plain"][:, :5])
        assert np.linalg.svd(q1.T @ q2, compute_uv=False).min() >= 1 - 1e-10
