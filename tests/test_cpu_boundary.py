"""CPU-only checks of the drop-in boundary: the C-ABI library loads and exports
every symbol declared in include/speclust_b200.h, the ctypes signature table
matches the header, host-side configuration / type validation mirrors the
reference, and the product path refuses to run without a GPU (no fallback)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1802_04450_b200 as sc
from paper_1802_04450_b200 import _native as nat
from paper_1802_04450_b200.errors import BadConfig, DimensionMismatch, InvalidFormat

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "speclust_b200.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = nat.load()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_signature_table_covers_header():
    assert set(header_symbols()) == set(nat.SIGNATURES), set(header_symbols()) ^ set(nat.SIGNATURES)


def test_version_callable_without_gpu():
    assert nat.load().sc_version() >= 100


def test_public_api_matches_reference_names():
    expected = {
        "CooMatrix", "CsrMatrix", "coo_canonicalize", "coo_to_csr", "csr_to_coo", "spmv",
        "SimilarityMeasure", "similarity", "build_edges_eps", "build_edges_knn", "build_edges_threshold",
        "build_similarity", "degrees", "handle_isolated", "row_scale", "sym_scale", "recover_row_eigvecs",
        "LanczosConfig", "EigenBasis", "rci_new", "rci_advance", "rci_extract", "eigensolve", "KmeansConfig",
        "Labeling", "pairwise_sq_dist", "kmeanspp_init", "lloyd", "kmeans", "cut", "ratio_cut", "ncut",
        "adjusted_rand_index", "PointsInput", "MatrixInput", "EdgesInput", "PipelineConfig", "ClusterReport",
        "run", "errors",
    }
    assert expected <= set(sc.__all__)
    for name in expected:
        assert hasattr(sc, name)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = sc.CsrMatrix(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(nat.NativeUnavailable):
        sc.spmv(m, np.ones(2))
    with pytest.raises(nat.NativeUnavailable):
        sc.degrees(m)


def test_status_codes_map_to_reference_errors():
    assert nat._STATUS[-1] is BadConfig
    assert nat._STATUS[-2] is DimensionMismatch
    assert nat._STATUS[-5] is sc.errors.NotSymmetric
    assert nat._STATUS[-9] is sc.errors.MaxRestartsExceeded


class TestHostTypes:
    def test_csr_validation(self):
        with pytest.raises(InvalidFormat):
            sc.CsrMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])
        with pytest.raises(InvalidFormat):
            sc.CsrMatrix(1, 3, [0, 2], [2, 0], [1.0, 1.0])
        with pytest.raises(InvalidFormat):
            sc.CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])

    def test_csr_arrays_read_only(self):
        m = sc.CsrMatrix(1, 1, [0, 1], [0], [5.0])
        with pytest.raises(ValueError):
            m.vals[0] = 1.0

    def test_canonicalize_and_convert(self):
        m = sc.coo_canonicalize(sc.CooMatrix(3, 3, [1, 0, 2, 1], [0, 1, 1, 2], [2.0, 2.0, 4.0, 4.0]))
        c = sc.coo_to_csr(m)
        assert list(c.row_ptr) == [0, 1, 3, 4]
        back = sc.csr_to_coo(c)
        assert np.array_equal(back.rows, m.rows) and np.array_equal(back.cols, m.cols)

    def test_duplicate_policy(self):
        with pytest.raises(sc.errors.DuplicateEntry):
            sc.coo_canonicalize(sc.CooMatrix(1, 1, [0, 0], [0, 0], [1.0, 2.0]), "error")
        assert sc.coo_canonicalize(sc.CooMatrix(1, 1, [0, 0], [0, 0], [1.0, 2.0])).vals[0] == 3.0


class TestConfigs:
    def test_kmeans_config(self):
        for bad in (dict(k=0), dict(k=2, max_iters=0), dict(k=2, tol_changes=-1), dict(k=2, init="x"),
                    dict(k=2, restarts=0)):
            with pytest.raises(BadConfig):
                sc.KmeansConfig(**bad)

    def test_measure(self):
        with pytest.raises(ValueError):
            sc.SimilarityMeasure.exp_decay(0.0)
        with pytest.raises(ValueError):
            sc.SimilarityMeasure("nope")
        assert sc.SimilarityMeasure.exp_decay(3.0).two_sigma_sq() == 18.0

    def test_pipeline_config(self):
        pin = sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(1.0), pattern="knn", points=np.zeros((3, 1)),
                             knn=1)
        with pytest.raises(BadConfig):
            sc.PipelineConfig(input=pin, k_clusters=1)
        with pytest.raises(BadConfig):
            sc.PipelineConfig(input=pin, k_clusters=2, eigen=sc.LanczosConfig(k=3))
        with pytest.raises(BadConfig):
            sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(1.0), pattern="knn", points=np.zeros((3, 1)))

    def test_similarity_scalar(self):
        m = sc.SimilarityMeasure.exp_decay(2.0)
        assert sc.similarity([0.0, 0.0], [3.0, 0.0], m) == pytest.approx(np.exp(-9.0 / 8.0))


def test_ari_host():
    assert sc.adjusted_rand_index([0, 0, 1, 1], [1, 1, 0, 0]) == 1.0
    assert sc.adjusted_rand_index([], []) == 1.0
