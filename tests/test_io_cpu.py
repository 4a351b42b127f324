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


_REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(_REF), reason="reference tree not present (build container only)")
def test_text_io_matches_reference_module(tmp_path):
    """Byte-identical files and identical parses / error classes against the
    reference's own io module (io.py:32-134), incl. extreme doubles and
    malformed inputs."""
    import importlib
    import sys

    sys.path.insert(0, _REF)
    try:
        rio = importlib.import_module("speclust.io")
        rsp = importlib.import_module("speclust.sparse")
    finally:
        sys.path.remove(_REF)
    rng = np.random.default_rng(7)
    vals = np.concatenate([rng.standard_normal(30) * 10.0 ** rng.integers(-300, 300, 30),
                           [5e-324, -0.0, 1.7976931348623157e308, 0.1, 1e16, 123456789.0]])
    n = 12
    rows, cols = rng.integers(0, n, len(vals)), rng.integers(0, n, len(vals))
    ours = sc.CooMatrix(n, n, rows, cols, vals)
    theirs = rsp.CooMatrix(n, n, rows, cols, vals)
    io.save_matrix(tmp_path / "a.txt", ours)
    rio.save_matrix(tmp_path / "b.txt", theirs)
    assert (tmp_path / "a.txt").read_bytes() == (tmp_path / "b.txt").read_bytes()
    got, want = io.load_matrix(tmp_path / "b.txt"), rio.load_matrix(tmp_path / "b.txt")
    assert np.array_equal(got.rows, want.rows) and np.array_equal(got.cols, want.cols)
    assert got.vals.tobytes() == want.vals.tobytes()
    x = vals[:36].reshape(6, 6)
    io.save_dense(tmp_path / "x1.txt", x)
    rio.save_dense(tmp_path / "x2.txt", x)
    assert (tmp_path / "x1.txt").read_bytes() == (tmp_path / "x2.txt").read_bytes()
    assert io.load_dense(tmp_path / "x2.txt").tobytes() == rio.load_dense(tmp_path / "x2.txt").tobytes()
    for fn_ours, fn_ref, arr in ((io.save_labels, rio.save_labels, rng.integers(-5, 9, 20)),
                                 (io.save_edges, rio.save_edges, rng.integers(0, 9, (7, 2)))):
        fn_ours(tmp_path / "o.txt", arr)
        fn_ref(tmp_path / "r.txt", arr)
        assert (tmp_path / "o.txt").read_bytes() == (tmp_path / "r.txt").read_bytes()
    bad = {"m_short.txt": ("load_matrix", "3 3 2\n0 1 0.5\n"), "m_tok.txt": ("load_matrix", "3 3 1\n0 1\n"),
           "m_hdr.txt": ("load_matrix", "3 3\n"), "d_row.txt": ("load_dense", "2 2\n1 2\n3\n"),
           "d_hdr.txt": ("load_dense", "2\n"), "e_bad.txt": ("load_edges", "0 1\n\n2 3 4\n"),
           "e_empty.txt": ("load_edges", "\n\n"), "l_blank.txt": ("load_labels", "1\n\n2\n")}
    for name, (fn, text) in bad.items():
        (tmp_path / name).write_text(text)
        outs = []
        for mod in (io, rio):
            try:
                r = getattr(mod, fn)(tmp_path / name)
                outs.append(("ok", np.asarray(getattr(r, "vals", r)).tolist()))
            except Exception as e:  # noqa: BLE001 - the class name and message are the contract
                outs.append((type(e).__name__, str(e)))
        assert outs[0] == outs[1], name
