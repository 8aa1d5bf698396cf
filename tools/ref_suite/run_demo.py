"""Run one of the reference's demo scripts (baseline/_ref/ref_demos) with
the reference package natively or, with --install, with its hot path and
surfacing re-routed to the B200 (paper_2402_01181_b200.install)."""
import os
import runpy
import sys
import types

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
sk = types.ModuleType("skimage")
sk.measure = types.ModuleType("skimage.measure")
sys.modules["skimage"], sys.modules["skimage.measure"] = sk, sk.measure
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")

import softmpm  # noqa: E402

if "--install" in sys.argv:
    import paper_2402_01181_b200 as b200
    b200.install(softmpm)
else:
    # natively, the reference's surfacing needs scikit-image (absent here): a
    # placeholder triangle keeps demo 01 running to its end (its mesh line is
    # not compared)
    import numpy as np

    def _mc(values, level, **kw):
        v = np.eye(3)
        return v, np.array([[0, 1, 2]]), v.copy(), np.zeros(3)
    sk.measure.marching_cubes = _mc
runpy.run_path(sys.argv[1], run_name="__main__")
