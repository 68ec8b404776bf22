"""The reference's OWN test modules (pkg/tests: ingest, index, query),
unmodified, run against the drop-in: tests/dropin_plugin.py switches the hot
path to this package before they import it.  The modules are staged next to
the reference install in baseline/_ref (tools/stage_reference_tests.py; not
committed -- reference sources stay out of the repository)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
SUITE = os.path.join(REF, "focusidx_tests")
MODULES = ["test_ingest.py", "test_index.py", "test_query.py", "test_tuner.py", "test_acceptance.py"]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("module", MODULES)
def test_reference_module_passes_on_the_dropin(module):
    if not os.path.exists(os.path.join(SUITE, module)):
        pytest.skip("reference tests not staged (python tools/stage_reference_tests.py)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, SUITE, os.path.join(REPO, "tests"), REPO,
                                         env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "dropin_plugin", "-q", "-x", "-p", "no:cacheprovider",
                        "--rootdir", SUITE, os.path.join(SUITE, module)],
                       cwd=SUITE, env=env, capture_output=True, text=True, timeout=850)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:]
