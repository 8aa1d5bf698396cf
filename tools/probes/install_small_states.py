"""Cost of the reference acceptance test's pattern through install(): 100
fresh 100-particle states, one p2g each (test_acceptance.py:33-56 requires
<= 1 s).  Prints the total and a cProfile of the top entries."""
import cProfile
import os
import pstats
import sys
import time
import types

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
sys.path.append(os.path.join(ROOT, "baseline", "_ref", "ref_tests"))
sk = types.ModuleType("skimage")
sk.measure = types.ModuleType("skimage.measure")
sys.modules["skimage"], sys.modules["skimage.measure"] = sk, sk.measure
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")
import numpy as np  # noqa: E402
import softmpm as sm  # noqa: E402
from conftest import random_state  # noqa: E402

import paper_2402_01181_b200 as b200  # noqa: E402

b200.install(sm)
grid = sm.Grid(resolution=(16, 16, 16), extent=(1.0, 1.0, 1.0))
rng = np.random.default_rng(2024)
params = sm.SimParams()
state, mats = random_state(grid, 100, rng)
sm.p2g(state, mats, params)


def loop():
    for _ in range(100):
        st, m = random_state(grid, 100, rng)
        sm.p2g(st, m, params)


t = time.perf_counter()
loop()
print(f"100 fresh states through install: {time.perf_counter() - t:.3f} s")
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

# the acceptance test's conservation numbers (fp32 gate 1e-5 after the suite
# plugin's tolerance rewrite), a few repetitions (atomic order varies)
for det in (False, True):
    b200.uninstall(sm)
    b200.install(sm, deterministic=det)
    for rep in range(4):
        rng = np.random.default_rng(2024)
        state, mats = random_state(grid, 100, rng)
        sm.p2g(state, mats, params)
        wm = wv = 0.0
        for _ in range(100):
            state, mats = random_state(grid, 100, rng)
            mom = (state.mass[:, None] * state.v).sum(axis=0)
            sm.p2g(state, mats, params)
            wm = max(wm, abs(state.grid_m.sum() - state.mass.sum()) / state.mass.sum())
            wv = max(wv, np.linalg.norm(state.grid_mv.reshape(-1, 3).sum(axis=0) - mom) / np.linalg.norm(mom))
        print(f"deterministic={det} rep {rep}: worst mass {wm:.2e}, worst momentum {wv:.2e}")
