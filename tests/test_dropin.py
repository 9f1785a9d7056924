"""The reference's own hot-path tests, unmodified, against the drop-in.

``dropin/sarfista`` is the reference package with its hot path (solver,
kernels seam, geometry, dictionary, rng) served by this engine and everything
else loaded from the installed reference (tools/install_reference.sh puts the
package in baseline/_ref and its test suite in baseline/_ref_tests; both
git-ignored, both travel to the GPU box).  Each case runs one reference test
file in a subprocess with ``PYTHONPATH=dropin`` and requires it to pass.

Not run: the reference's CLI, experiment-harness, image-IO and sampling test
files (out of scope; they exercise reference code only), and the
acceptance criteria that run the desk-scale experiment grid end to end
(5-8, 11: preset sweeps through the reference harness, minutes each).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(REPO, "baseline", "_ref_tests")
REPORT = os.environ.get("SF_DROPIN_REPORT")

CASES = [
    ("test_solver.py", None),
    ("test_kernels.py", None),
    ("test_geometry.py", None),
    ("test_dictionary.py", None),
    ("test_rng.py", None),
    ("test_acceptance.py", "criterion_01 or criterion_02 or criterion_03 or criterion_04 "
                           "or criterion_09 or criterion_10"),
]


@pytest.mark.parametrize("name,select", CASES, ids=[c[0] for c in CASES])
def test_reference_suite_passes_against_dropin(name, select):
    if not os.path.isfile(os.path.join(REF_TESTS, name)):
        pytest.skip("reference tests not installed (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "dropin"), REPO,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-rs", name]
    if select:
        cmd += ["-k", select]
    proc = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True,
                          timeout=1800)
    tail = "\n".join(proc.stdout.strip().splitlines()[-15:])
    print(f"DROPIN {name}: rc={proc.returncode}\n{tail}")
    if REPORT:
        with open(REPORT, "a") as fh:
            fh.write(f"== {name} (-k {select!r}) rc={proc.returncode}\n{proc.stdout}\n")
    assert proc.returncode == 0, proc.stdout[-4000:] + proc.stderr[-2000:]
