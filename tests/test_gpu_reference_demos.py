"""The reference's demo scripts (pkg/demos/01_elastic_block.py,
02_tool_contact.py, 03_stiffness_sweep.py -- copied unmodified into
baseline/_ref/ref_demos by tools/install_reference.sh) run natively (numba
CPU) and through install() (B200); every number they print must agree to
fp32 tolerance, except wall-clock timings and demo 01's mesh size (the
native run has no scikit-image here)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMOS = os.path.join(ROOT, "baseline", "_ref", "ref_demos")
RUN = os.path.join(ROOT, "tools", "ref_suite", "run_demo.py")
NUM = re.compile(r"[-+]?\d+\.?\d*(?:[eE][-+]?\d+)?")


def _run(demo, install, tmp):
    env = dict(os.environ)
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")
    args = [sys.executable, RUN, os.path.join(DEMOS, demo)] + (["--install"] if install else [])
    r = subprocess.run(args, cwd=tmp, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return r.stdout


def _numbers(out):
    rows = []
    for ln in out.splitlines():
        if ln.startswith("wrote "):  # demo 01's mesh: native run has no scikit-image here
            continue
        ln = re.sub(r"soft=[0-9.]+ ms", "", ln)  # wall-clock timings
        rows.append([float(t) for t in NUM.findall(ln)])
    return rows


@pytest.mark.skipif(not os.path.isdir(DEMOS), reason="reference not installed (bash tools/install_reference.sh)")
@pytest.mark.parametrize("demo,rel", [("01_elastic_block.py", 1e-3), ("02_tool_contact.py", 2e-2),
                                      ("03_stiffness_sweep.py", 2e-2)])
def test_reference_demo_through_install(demo, rel, tmp_path):
    native = _run(demo, False, tmp_path)
    gpu = _run(demo, True, tmp_path)
    print("---- native\n" + native + "---- install()\n" + gpu)
    a, b = _numbers(native), _numbers(gpu)
    assert len(a) == len(b)
    for ra, rb in zip(a, b):
        assert len(ra) == len(rb)
        for x, y in zip(ra, rb):
            assert abs(x - y) <= rel * max(abs(x), abs(y)) + 2e-3, (x, y, demo)
