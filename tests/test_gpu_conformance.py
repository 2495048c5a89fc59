"""GPU: the reference's own test suite (in-scope modules) through the `defcg`
shim (conformance/).  The reference's test files are
staged by `python tools/conformance.py stage` in the build container into the
git-ignored conformance/_reftests/ (they travel with the repo snapshot);
without the staged copy this test is skipped."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
STAGE = ROOT / "conformance" / "_reftests"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not STAGE.exists(), reason="reference tests not staged (tools/conformance.py stage)")
def test_reference_suite_passes_through_shim():
    res = subprocess.run([sys.executable, str(ROOT / "tools" / "conformance.py"), "run", "-q", "--tb=short"],
                         capture_output=True, text=True, timeout=1800)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
