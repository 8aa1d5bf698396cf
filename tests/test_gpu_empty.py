"""Empty particle sets (an edge case the reference accepts: core.step over
zero particles runs the grid ops on an empty grid and advances the clock,
core.py:280-320; its stage functions are no-ops).  The drop-in matches that
through the C ABI (an uploaded empty set is valid state), and a state that
later gains particles steps normally."""
import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import scenes

pytestmark = pytest.mark.gpu


def _empty(res=32):
    grid = sm.Grid((res, res, res))
    z3, z33 = np.zeros((0, 3)), np.zeros((0, 3, 3))
    st = sm.SimState(grid, z3, z3, z33, z33, np.zeros(0), np.zeros(0), np.zeros(0, np.int32))
    return grid, st, [sm.Material(1.0e4, 0.3, 1000.0)]


def test_empty_state_step_and_stages():
    grid, st, mats = _empty()
    params = sm.SimParams()
    rep = sm.step(st, mats, params)
    assert rep.inverted_particles == 0 and st.step_count == 1
    assert st.time == pytest.approx(params.substeps_per_frame * params.dt, rel=1e-12)
    assert st.x.shape == (0, 3) and st.F.shape == (0, 3, 3)
    assert not st.has_nan()
    assert not st.grid_m.any() and not st.grid_mv.any()
    assert sm.p2g(st, mats, params) == 0
    assert not st.grid_m.any()
    sm.grid_update(st, params)
    sm.g2p_advect(st, params)
    assert sm.substep(st, mats, params) == 0
    m = sm.compute_metrics(st, np.zeros((0, 3)))
    assert np.isnan(m.lifted_fraction)


def test_empty_state_with_tool_builds_the_collision_field():
    grid, st, mats = _empty()
    tool = sm.RigidCollider(id=0, shape=sm.Box([0.1, 0.05, 0.1]), translation=[0.5, 0.5, 0.5])
    sm.step(st, mats, sm.SimParams(), [tool])
    cf = st._collision
    assert cf is not None and (cf.object_id == 0).sum() > 0  # nodes within 2 theta of the box


def test_empty_state_then_particles():
    grid, st, mats = _empty(64)
    sm.step(st, mats, sm.SimParams())
    ref, _, params, _, _ = scenes.c1(count=2000, res=64)
    st.x, st.v, st.F, st.C = ref.x, ref.v, ref.F, ref.C
    st.mass, st.vol0, st.material_id = ref.mass, ref.vol0, ref.material_id
    sm.step(st, mats, params)
    sm.step(ref, mats, params)
    assert np.allclose(st.x, ref.x, rtol=0, atol=1e-6)
