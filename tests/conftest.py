import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)


def packed_from_golden(g, prefix="col"):
    from paper_2402_01181_b200.collision import PackedColliders
    keys = ["kind", "half", "rotation", "translation", "linear_velocity", "angular_velocity",
            "friction", "mode", "sdf_values", "sdf_offset", "sdf_resolution",
            "sdf_bounds_min", "sdf_extent"]
    return PackedColliders(*[np.array(g[f"{prefix}_{k}"]) for k in keys])
