"""The reference package's OWN hot-path tests, run through install().

tools/install_reference.sh installs the unmodified reference (softmpm) into
baseline/_ref and copies its tests/test_transfers.py, test_substep.py,
test_collision.py, test_weights.py, test_materials.py and test_oracle.py
(/root/reference/pkg/tests) beside it.  tools/ref_suite/ref_suite_plugin.py
imports that softmpm, calls paper_2402_01181_b200.install(softmpm) -- so
softmpm.p2g / grid_update / g2p_advect / substep / step run on the B200
kernels -- and maps the tests' fp64 tolerance literals (< 1e-5 on the right
of a < / <= comparison or as an approx / allclose tolerance) to the fp32
gate 1e-5.  The test runs that suite in a subprocess and requires every test
to pass except the ones listed in EXPECTED_FAIL with the reason."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
MODULES = ["test_transfers.py", "test_substep.py", "test_collision.py", "test_weights.py",
           "test_materials.py", "test_oracle.py"]
# test id -> why it cannot hold for the fp32 drop-in (documented in DESIGN.md)
EXPECTED_FAIL: dict[str, str] = {}


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "ref_tests")),
                    reason="reference not installed (bash tools/install_reference.sh)")
def test_reference_hot_path_suite_through_install():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tools", "ref_suite"), REF, ROOT,
                                         env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")
    files = [os.path.join(REF, "ref_tests", m) for m in MODULES]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-rA", "-p", "ref_suite_plugin",
                        "-p", "no:cacheprovider", "--rootdir", os.path.join(REF, "ref_tests"), *files],
                       cwd=os.path.join(REF, "ref_tests"), env=env, capture_output=True, text=True,
                       timeout=1200)
    out = r.stdout + r.stderr
    print(out[-8000:])
    assert "install() active: True" in out
    failed = [ln.split()[1] for ln in out.splitlines() if ln.startswith("FAILED ")]
    failed = [f.split("::", 1)[1] if "::" in f else f for f in failed]
    unexpected = [f for f in failed if f not in EXPECTED_FAIL]
    assert not unexpected, unexpected
    assert " passed" in out
