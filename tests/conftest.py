"""Shared pytest configuration.

Markers:
  gpu  -- needs a CUDA device and the built libspeclust_b200.so (run on the
          B200 box with ``pytest -m gpu``); everything else runs on CPU.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200) and the native library")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz") as f:
                cache[name] = {k: f[k] for k in f.files}
        return cache[name]

    return load
