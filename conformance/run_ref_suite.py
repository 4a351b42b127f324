"""Conformance run of the reference package's OWN test suite against this
engine (the reference tests are a free drop-in check).

    python conformance/run_ref_suite.py --stage   # build container: copy the suite
    python conformance/run_ref_suite.py           # GPU box: run it, write the report

``--stage`` copies /root/reference/pkg/tests/*.py (minus test_cli.py: the CLI
is out of scope) into conformance/ref_suite/ -- git-ignored, so no reference
source enters the history, but shipped to the GPU box with the snapshot.  The
run aliases ``speclust`` and its submodules to ``paper_1802_04450_b200`` in a
generated conftest, deselects the reference's ``slow`` marker and writes a
junit + summary report.  It lives outside tests/ on purpose: reference tests
that pin numpy-stream-specific outputs (e.g. the SBM generator's exact draws)
are expected to differ and must not break the product test run."""
from __future__ import annotations

import argparse
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SUITE = HERE / "ref_suite"
REF_TESTS = Path("/root/reference/pkg/tests")

CONFTEST = '''"""Generated: alias speclust -> paper_1802_04450_b200 for the reference suite."""
import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
pkg = importlib.import_module("paper_1802_04450_b200")
sys.modules["speclust"] = pkg
for sub in ("sparse", "graph", "laplacian", "eigen", "kmeans", "metrics", "pipeline", "errors", "io", "sbm"):
    sys.modules["speclust." + sub] = importlib.import_module("paper_1802_04450_b200." + sub)

# the CLI is out of scope (SURVEY.md §8): tests that drive it are skipped
import types  # noqa: E402

import pytest  # noqa: E402


def _cli_main(*a, **k):
    pytest.skip("speclust.cli is out of scope for this engine")


_cli = types.ModuleType("speclust.cli")
_cli.main = _cli_main
sys.modules["speclust.cli"] = _cli


def pytest_configure(config):
    config.addinivalue_line("markers", "slow: heavy optional workload (reference marker)")
'''


def stage():
    if not REF_TESTS.is_dir():
        sys.exit(f"{REF_TESTS} not found (stage in the build container)")
    SUITE.mkdir(exist_ok=True)
    for p in sorted(REF_TESTS.glob("*.py")):
        if p.name == "test_cli.py":
            continue
        shutil.copy(p, SUITE / p.name)
    (SUITE / "conftest.py").write_text(CONFTEST)
    print(f"staged {len(list(SUITE.glob('test_*.py')))} test files into {SUITE}")


def run(out_dir: Path):
    out_dir.mkdir(parents=True, exist_ok=True)
    junit = out_dir / "ref_suite_junit.xml"
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-m", "not slow", "-p", "no:cacheprovider",
           f"--junitxml={junit}", "--rootdir", str(SUITE)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    (out_dir / "ref_suite.log").write_text(res.stdout + res.stderr)
    print("\n".join(res.stdout.strip().splitlines()[-40:]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true")
    ap.add_argument("--out", default="gpurun_out")
    a = ap.parse_args()
    stage() if a.stage else run(Path(a.out))
