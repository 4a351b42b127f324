"""Device loading of binary CSR containers: every CSR invariant the device
kernels rely on is validated (sc_csr_validate) before a DeviceCsr is handed
out (sparse.py:83-142 checks, applied to untrusted .scb input)."""

import numpy as np
import pytest

import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import io

pytestmark = pytest.mark.gpu


def _write(path, n_rows, n_cols, rp, col, vals, isz=4):
    with open(path, "wb") as f:
        f.write(b"SCB1CSR\0")
        np.array([n_rows, n_cols, len(vals), isz], dtype="<i8").tofile(f)
        np.asarray(rp, dtype="<i8").tofile(f)
        np.asarray(col, dtype=np.int32 if isz == 4 else np.int64).tofile(f)
        np.asarray(vals, dtype="<f8").tofile(f)


def test_valid_container_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    a = (rng.random((300, 300)) < 0.05) * rng.standard_normal((300, 300))
    r, c = np.nonzero(a)
    m = sc.coo_to_csr(sc.coo_canonicalize(sc.CooMatrix(300, 300, r, c, a[r, c])))
    io.save_csr_binary(tmp_path / "m.scb", m)
    d = io.load_csr_binary(tmp_path / "m.scb", device=True)
    h = d.to_host()
    assert np.array_equal(h.row_ptr, m.row_ptr) and np.array_equal(h.col_idx, m.col_idx)
    assert h.vals.tobytes() == m.vals.tobytes()


@pytest.mark.parametrize("case", ["rp_start", "rp_end", "rp_decrease", "col_range", "col_order", "col_dup",
                                  "nan", "col64_range"])
def test_malformed_container_rejected(tmp_path, case):
    rp, col, vals = [0, 2, 3, 5], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0]
    isz = 4
    if case == "rp_start":
        rp = [1, 2, 3, 5]
    elif case == "rp_end":
        rp = [0, 2, 3, 4]
    elif case == "rp_decrease":
        rp = [0, 3, 2, 5]
    elif case == "col_range":
        col = [0, 2, 1, 0, 3]
    elif case == "col_order":
        col = [2, 0, 1, 0, 2]
    elif case == "col_dup":
        col = [0, 2, 1, 2, 2]
    elif case == "nan":
        vals = [1.0, np.nan, 3.0, 4.0, 5.0]
    elif case == "col64_range":
        col, isz = [0, 2, 1, 0, 2**33], 8
    _write(tmp_path / "bad.scb", 3, 3, rp, col, vals, isz)
    with pytest.raises(sc.errors.InvalidFormat):
        io.load_csr_binary(tmp_path / "bad.scb", device=True)
    with pytest.raises(sc.errors.InvalidFormat):
        io.load_csr_binary(tmp_path / "bad.scb", device=False)
