"""File formats: the reference's text formats and the
binary containers, CPU only (no device calls)."""

import numpy as np
import pytest

import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import io


def _csr(rng, n=40, dens=0.1):
    a = (rng.random((n, n)) < dens) * rng.standard_normal((n, n))
    r, c = np.nonzero(a)
    return sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(n, n, r, c, a[r, c])))


def test_text_round_trips_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    m = _csr(rng)
    io.save_matrix(tmp_path / "m.txt", m)
    back = io.load_matrix(tmp_path / "m.txt")
    assert back.n_rows == m.n_rows and np.array_equal(back.vals, m.vals)
    assert np.array_equal(back.rows, m.row_indices()) and np.array_equal(back.cols, m.col_idx)
    x = rng.standard_normal((7, 3)) * 1e-300
    io.save_dense(tmp_path / "x.txt", x)
    assert np.array_equal(io.load_dense(tmp_path / "x.txt"), x)
    assert np.array_equal(io.load_points(tmp_path / "x.txt"), x)
    lab = rng.integers(0, 9, 50)
    io.save_labels(tmp_path / "l.txt", lab)
    assert np.array_equal(io.load_labels(tmp_path / "l.txt"), lab)
    e = np.array([[0, 3], [2, 5], [1, 4]])
    io.save_edges(tmp_path / "e.txt", e)
    assert np.array_equal(io.load_edges(tmp_path / "e.txt"), e)


def test_text_format_matches_reference_layout(tmp_path):
    # header `n_rows n_cols nnz`, entries `row col repr(value)` (io.py:32-44)
    m = sc.coo_to_csr(sc.CooMatrix(3, 3, [0, 2], [1, 0], [0.1, -2.5]))
    io.save_matrix(tmp_path / "m.txt", m)
    assert (tmp_path / "m.txt").read_text() == "3 3 2\n0 1 0.1\n2 0 -2.5\n"
    (tmp_path / "bad.txt").write_text("3 3\n")
    with pytest.raises(sc.errors.InvalidFormat):
        io.load_matrix(tmp_path / "bad.txt")
    (tmp_path / "nan.txt").write_text("1 2\nnan 1.0\n")
    with pytest.raises(sc.errors.InvalidFormat):
        io.load_points(tmp_path / "nan.txt")


def test_binary_containers(tmp_path):
    rng = np.random.default_rng(1)
    m = _csr(rng, 300, 0.05)
    io.save_csr_binary(tmp_path / "m.scb", m)
    back = io.load_csr_binary(tmp_path / "m.scb")
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.col_idx, m.col_idx)
    assert np.array_equal(back.vals, m.vals)
    x = rng.standard_normal((11, 5))
    io.save_dense_binary(tmp_path / "x.scb", x)
    assert np.array_equal(io.load_dense_binary(tmp_path / "x.scb"), x)
    lab = rng.integers(0, 100, 1000)
    io.save_labels_binary(tmp_path / "l.scb", lab)
    assert np.array_equal(io.load_labels_binary(tmp_path / "l.scb"), lab)
    with pytest.raises(sc.errors.InvalidFormat):
        io.load_dense_binary(tmp_path / "l.scb")  # wrong container kind
    (tmp_path / "t.scb").write_bytes((tmp_path / "m.scb").read_bytes()[:100])
    with pytest.raises(sc.errors.InvalidFormat):
        io.load_csr_binary(tmp_path / "t.scb")


def test_sbm_config_validation():
    with pytest.raises(sc.errors.BadConfig):
        sc.SbmConfig(block_sizes=(), p_in=0.5, p_out=0.1)
    with pytest.raises(sc.errors.BadConfig):
        sc.SbmConfig(block_sizes=(10, 0), p_in=0.5, p_out=0.1)
    with pytest.raises(sc.errors.BadConfig):
        sc.SbmConfig(block_sizes=(10, 10), p_in=0.1, p_out=0.5)
    assert sc.SbmConfig(block_sizes=[3, 4], p_in=0.5, p_out=0.1).block_sizes == (3, 4)
