"""GPU parity of the frame consumers: density splat and metrics
through the C ABI against the oracle restatement / reference golden vectors
(tests/golden/frame_ops.npz), plus the reference's own test cases
(tests/test_surfacing.py:16-37, tests/test_scene.py:154-185).

Tolerances: splat with fp64 positions uses fp64 weights and fp64 atomics, so
it differs from the chunk-ordered reference only by summation order
(rel 1e-12 of the field maximum); the device state is fp32, so metrics on it
carry fp32 rounding of x and F (rel 1e-5 on mean |J - 1|, 1e-6 on
displacements)."""
import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from conftest import load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _blob_state(g):
    grid = sm.Grid((16, 16, 16), (1.0, 1.0, 1.0))
    n = len(g["blob_x"])
    return sm.SimState(grid, g["blob_x"], np.zeros((n, 3)), np.tile(np.eye(3), (n, 1, 1)),
                       np.zeros((n, 3, 3)), g["blob_mass"], g["blob_mass"] / 1000.0, np.zeros(n, np.int32))


def test_splat_density_matches_reference():
    g = load_golden("frame_ops.npz")
    grid = sm.Grid((16, 16, 16), (1.0, 1.0, 1.0))
    for key, res in (("splat16", None), ("splat32", (32, 32, 32))):
        fld = sm.splat_density(g["blob_x"], g["blob_mass"], grid, res)
        ref = g[key]
        assert fld.values.shape == ref.shape
        assert fld.dx == pytest.approx(float(g[f"{key}_dx"]), rel=1e-15)
        assert np.abs(fld.values - ref).max() <= 1e-12 * ref.max(), key


def test_density_field_from_device_state():
    g = load_golden("frame_ops.npz")
    st = _blob_state(g)
    fld = sm.density_field(st, (32, 32, 32))
    x32 = g["blob_x"].astype(np.float32).astype(np.float64)
    m32 = g["blob_mass"].astype(np.float32).astype(np.float64)
    ref = O.splat_density(x32, m32, (32, 32, 32), 1.0 / 32)
    assert np.abs(fld.values - ref).max() <= 1e-12 * ref.max()
    # mass conservation (tests/test_surfacing.py:16-21)
    assert fld.values.sum() * fld.dx ** 3 == pytest.approx(m32.sum(), rel=1e-12)
    assert (fld.values >= 0.0).all()


def test_splat_empty_and_single_particle():
    grid = sm.Grid((16, 16, 16), (1.0, 1.0, 1.0))
    assert np.abs(sm.splat_density(np.zeros((0, 3)), np.zeros(0), grid).values).max() == 0.0
    x = np.array([[0.5, 0.5, 0.5]])
    fld = sm.splat_density(x, np.array([1.0e-3]), grid)
    base, _ = sm.bspline_weights(x[0], grid)
    nz = np.argwhere(fld.values > 0.0)
    assert len(nz) <= 27
    assert (nz.min(axis=0) >= base).all() and (nz.max(axis=0) <= base + 2).all()


def test_compute_metrics_matches_reference():
    g = load_golden("frame_ops.npz")
    grid = sm.Grid((32, 32, 32), (1.0, 1.0, 1.0))
    n = len(g["met_x"])
    st = sm.SimState(grid, g["met_x"], np.zeros((n, 3)), g["met_F"], np.zeros((n, 3, 3)), np.full(n, 1e-3),
                     np.full(n, 1e-6), np.zeros(n, np.int32))
    m = sm.compute_metrics(st, g["met_x0"])
    ref = g["met"]
    assert m.lifted_fraction == pytest.approx(ref[0], abs=1.0 / n)
    assert m.detached_fraction == pytest.approx(ref[1], abs=1.0 / n)
    assert m.mean_abs_j_minus_1 == pytest.approx(ref[2], rel=1e-5)
    assert m.max_displacement == pytest.approx(ref[3], rel=1e-6)
    # second call reuses the uploaded reference positions
    m2 = sm.compute_metrics(st, g["met_x0"])
    assert m2 == m


def test_compute_metrics_reference_cases():
    grid = sm.Grid((16, 16, 16), (1.0, 1.0, 1.0))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.4, 0.5), (0.3, 0.2, 0.3), 500, seed=8, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    x0 = st.x.copy()
    m = sm.compute_metrics(st, x0)
    assert (m.lifted_fraction, m.detached_fraction, m.mean_abs_j_minus_1) == (0.0, 0.0, 0.0)
    assert m.max_displacement < 1e-7
    st.x[:, 1] += 5.0 * grid.dx
    m = sm.compute_metrics(st, x0)
    assert m.lifted_fraction == 1.0 and m.detached_fraction == 1.0
    assert m.mean_abs_j_minus_1 < 1e-12
    assert m.max_displacement == pytest.approx(5.0 * grid.dx, rel=1e-6)
    st.F[:] = np.diag([0.9, 0.9, 0.9])
    m = sm.compute_metrics(st, st.x.copy())
    assert m.mean_abs_j_minus_1 == pytest.approx(1.0 - 0.729, rel=1e-6)


def test_metrics_after_gpu_frame_vs_oracle():
    """A device frame, then metrics on the device vs the oracle on the
    downloaded state."""
    grid = sm.Grid((32, 32, 32))
    mats = [sm.Material(1e4, 0.3, 1000.0)]
    st = sm.SimState.from_spawns(grid, [sm.sample_box((0.5, 0.14, 0.5), (0.3, 0.16, 0.3), 3000, seed=4,
                                                      grid=grid)], mats)
    x0 = st.x.copy()
    sm.step(st, mats, sm.SimParams())
    m = sm.compute_metrics(st, x0)
    ref = O.compute_metrics(st.x, st.F, x0, grid.dx)
    assert m.lifted_fraction == pytest.approx(ref[0], abs=1e-9)
    assert m.mean_abs_j_minus_1 == pytest.approx(ref[2], rel=1e-6)
    assert m.max_displacement == pytest.approx(ref[3], rel=1e-6)
