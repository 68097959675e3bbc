"""Run the REFERENCE's own test files against this package (import alias).

    python scripts/run_reference_tests.py prepare   # dev container (has /root/reference)
    python scripts/run_reference_tests.py run       # GPU box: pytest on the copies

``prepare`` copies ``/root/reference/pkg/tests/*.py`` and the reference's
test-only oracle module (``kcliques/oracle.py``: brute force, naive recursion,
matrix-trace triangles) into ``baseline/_ref_tests/`` -- git-ignored, never
committed, but shipped to the GPU box by gpurun -- and writes an alias package
``kcliques`` there whose public names are this package's (the GPU drop-in).
``run`` executes the reference's tests unchanged against that alias and
writes the junit/log under ``gpurun_out/``.  Tests that pin CPU
implementation details (the numba worker-scratch byte formula, per-thread
worker load lists) are expected to differ and are listed in the log summary.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DEST = os.path.join(REPO, "baseline", "_ref_tests")
REF = "/root/reference/pkg"

ALIAS = '''"""Import alias: the reference's tests see the B200 package as `kcliques`."""
import sys

import paper_2104_13209_b200 as _pkg
from paper_2104_13209_b200 import *  # noqa: F401,F403  the GPU drop-in
from paper_2104_13209_b200 import cli as _cli
from paper_2104_13209_b200 import orientation as _orientation

sys.modules[__name__ + ".orientation"] = _orientation
sys.modules[__name__ + ".cli"] = _cli
cli = _cli
# the reference's own test-only oracles (checkers, not the thing measured)
from .oracle import brute_force_count, naive_recursive_count, triangle_count  # noqa: E402,F401

__version__ = _pkg.__version__
'''


def prepare() -> None:
    if os.path.isdir(DEST):
        shutil.rmtree(DEST)
    os.makedirs(os.path.join(DEST, "tests"))
    os.makedirs(os.path.join(DEST, "kcliques"))
    for f in glob.glob(os.path.join(REF, "tests", "*.py")):
        shutil.copy(f, os.path.join(DEST, "tests"))
    shutil.copy(os.path.join(REF, "src", "kcliques", "oracle.py"),
                os.path.join(DEST, "kcliques", "oracle.py"))
    with open(os.path.join(DEST, "kcliques", "__init__.py"), "w") as f:
        f.write(ALIAS)
    print(f"prepared {DEST}")


def run() -> int:
    out = os.path.join(REPO, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([DEST, REPO, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", os.path.join(DEST, "tests"), "-q", "-rfE",
           "-p", "no:cacheprovider", "--junitxml", os.path.join(out, "ref_tests.xml")]
    r = subprocess.run(cmd, env=env, cwd=DEST, capture_output=True, text=True)
    with open(os.path.join(out, "ref_tests.log"), "w") as f:
        f.write(r.stdout + "\n" + r.stderr)
    print(r.stdout[-4000:])
    return r.returncode


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "prepare":
        prepare()
    else:
        sys.exit(run())
