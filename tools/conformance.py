"""Run the reference's own test suite against the B200 package through the
`defcg` shim in conformance/ (SURVEY.md section 4).

  python tools/conformance.py stage   # in the build container: copy the
                                      # reference's in-scope test files into
                                      # conformance/_reftests/ (git-ignored)
  python tools/conformance.py run [pytest args]   # on the GPU box
"""
import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STAGE = ROOT / "conformance" / "_reftests"
REF_TESTS = Path("/root/reference/pkg/tests")
IN_SCOPE = ["conftest.py", "test_solvers.py", "test_recycle.py", "test_gpc.py", "test_linalg.py",
            "test_kernels.py", "test_subset.py", "test_acceptance.py"]


def stage():
    STAGE.mkdir(parents=True, exist_ok=True)
    for name in IN_SCOPE:
        shutil.copy2(REF_TESTS / name, STAGE / name)
    (STAGE / "SOURCE.txt").write_text(f"copied from {REF_TESTS} by tools/conformance.py stage; not committed\n")
    print(f"staged {len(IN_SCOPE)} files into {STAGE}")


def run(args):
    if not STAGE.exists():
        sys.exit("conformance/_reftests is not staged (python tools/conformance.py stage, in the build container)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "conformance"), str(ROOT), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", str(STAGE), "-q", "-p", "no:cacheprovider", "--rootdir", str(STAGE),
           "-c", os.devnull, *args]
    return subprocess.call(cmd, env=env, cwd=str(STAGE))


if __name__ == "__main__":
    if len(sys.argv) < 2 or sys.argv[1] not in ("stage", "run"):
        sys.exit(__doc__)
    if sys.argv[1] == "stage":
        stage()
    else:
        sys.exit(run(sys.argv[2:]))
