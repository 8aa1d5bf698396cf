"""The reference's own behavioural test cases (tests/test_transfers.py,
tests/test_substep.py, tests/test_collision.py) restated against the CUDA
path.  Same setups and assertions; tolerances that the reference states for
fp64 numba code are widened to fp32 device state where noted (the device
keeps x, v, F, C in fp32: a host fp64 value round-trips with ~6e-8 relative
error, and fixed-point P2G adds ~1e-7 of the per-item bound)."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import paper_2402_01181_b200 as sm

pytestmark = pytest.mark.gpu

F32 = 1e-6  # relative tolerance for a single fp32 round trip / one substep


@pytest.fixture
def small_grid():
    return sm.Grid(resolution=(16, 16, 16), extent=(1.0, 1.0, 1.0))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_state(grid, n, rng, young=5.0e3, spread=0.2):
    """conftest.random_state: random-but-valid state for transfer tests."""
    materials = [sm.Material(young, 0.3, 1000.0)]
    lo, hi = grid.margin_bounds()
    x = rng.uniform(lo + spread * 0.1, hi - spread * 0.1, (n, 3))
    state = sm.SimState(grid=grid, x=x, v=rng.normal(0.0, 0.5, (n, 3)),
                        F=np.tile(np.eye(3), (n, 1, 1)) + rng.normal(0.0, 0.05, (n, 3, 3)),
                        C=rng.normal(0.0, 2.0, (n, 3, 3)), mass=rng.uniform(1.0e-4, 2.0e-3, n),
                        vol0=rng.uniform(1.0e-7, 1.0e-6, n), material_id=np.zeros(n, dtype=np.int32))
    return state, materials


def one_particle_state(grid, positions):
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.ParticleSpawn(positions=np.asarray(positions, dtype=np.float64), rest_volume_per_particle=1e-6,
                             material_id=0)
    return sm.SimState.from_spawns(grid, [spawn], mats), mats


# ---------------------------------------------------------------- transfers
def test_p2g_single_particle_at_rest(small_grid):
    """test_transfers.py:8-15: at rest the stress vanishes exactly, so the grid
    carries no momentum; the mass lands on the grid."""
    state, mats = one_particle_state(small_grid, [[0.43, 0.57, 0.5]])
    sm.p2g(state, mats, sm.SimParams())
    assert np.abs(state.grid_mv).max() == 0.0
    assert state.grid_m.sum() == pytest.approx(state.mass.sum(), rel=F32)


def test_p2g_conserves_mass_and_momentum(small_grid, rng):
    """test_transfers.py:18-29 (1e-9 in fp64; fixed-point fp32 here)."""
    params = sm.SimParams()
    for _ in range(20):
        state, mats = random_state(small_grid, 100, rng)
        momentum_before = (state.mass[:, None] * state.v).sum(axis=0)
        mass = state.mass.sum()
        sm.p2g(state, mats, params)
        assert abs(state.grid_m.sum() - mass) / mass < 1e-5
        grid_momentum = state.grid_mv.reshape(-1, 3).sum(axis=0)
        rel = np.linalg.norm(grid_momentum - momentum_before) / max(np.linalg.norm(momentum_before), 1e-30)
        assert rel < 1e-4


def test_p2g_reports_inverted_elements(small_grid):
    """test_transfers.py:32-40."""
    state, mats = one_particle_state(small_grid, [[0.5, 0.5, 0.5], [0.4, 0.4, 0.4]])
    state.F[0] = np.diag([-0.5, 1.0, 1.0])
    assert sm.p2g(state, mats, sm.SimParams()) == 1
    assert not state.has_nan()


def test_grid_update_momentum_to_velocity(small_grid):
    """test_transfers.py:43-57: mv / m, zero-mass nodes untouched (exact)."""
    state, _ = one_particle_state(small_grid, [[0.5, 0.5, 0.5]])
    state.grid_m[:] = 0.0
    state.grid_mv[:] = 0.0
    state.grid_m[8, 8, 8] = 2.0
    state.grid_mv[8, 8, 8] = (2.0, 0.0, 0.0)
    state.grid_m[4, 4, 4] = 0.0
    state.grid_mv[4, 4, 4] = (9.0, 9.0, 9.0)
    sm.grid_update(state, sm.SimParams(gravity=(0.0, 0.0, 0.0)))
    assert np.array_equal(state.grid_mv[8, 8, 8], (1.0, 0.0, 0.0))
    assert np.array_equal(state.grid_mv[4, 4, 4], (9.0, 9.0, 9.0))


def test_boundary_clamp_normal_only(small_grid):
    """test_transfers.py:60-71."""
    state, _ = one_particle_state(small_grid, [[0.5, 0.5, 0.5]])
    state.grid_m[:] = 0.0
    state.grid_mv[:] = 0.0
    state.grid_m[8, 1, 8] = 1.0
    state.grid_mv[8, 1, 8] = (0.3, -1.0, 0.0)
    sm.grid_update(state, sm.SimParams(gravity=(0.0, 0.0, 0.0)))
    assert np.allclose(state.grid_mv[8, 1, 8], (0.3, 0.0, 0.0), rtol=F32, atol=0.0)
    assert state.grid_mv[8, 1, 8][1] == 0.0


def test_boundary_stick_zeroes_all(small_grid):
    """test_transfers.py:74-84."""
    state, _ = one_particle_state(small_grid, [[0.5, 0.5, 0.5]])
    state.grid_m[:] = 0.0
    state.grid_mv[:] = 0.0
    state.grid_m[8, 1, 8] = 1.0
    state.grid_mv[8, 1, 8] = (0.3, -1.0, 0.2)
    sm.grid_update(state, sm.SimParams(gravity=(0.0, 0.0, 0.0), boundary="stick"))
    assert np.abs(state.grid_mv[8, 1, 8]).max() == 0.0


def test_g2p_reproduces_constant_field(small_grid, rng):
    """test_transfers.py:87-97."""
    state, _ = random_state(small_grid, 50, rng)
    state.C[:] = 0.0
    u = np.array([0.3, -0.2, 0.5])
    state.grid_mv[:] = u
    x_before = state.x.copy()
    params = sm.SimParams()
    sm.g2p_advect(state, params)
    assert np.abs(state.v - u).max() < 1e-6
    assert np.abs(state.C).max() < 1e-4  # |C| ~ 4/dx^2 * fp32 rounding of sum w v dp
    assert np.abs(state.x - (x_before + params.dt * u)).max() < 2e-7


def test_g2p_reproduces_affine_field(small_grid, rng):
    """test_transfers.py:100-113: APIC recovers v(x) = A x."""
    state, _ = random_state(small_grid, 50, rng)
    a = rng.normal(0.0, 1.0, (3, 3))
    nx, ny, nz = small_grid.resolution
    nodes = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"),
                     axis=-1) * small_grid.dx
    state.grid_mv[:] = nodes @ a.T
    x_before = state.x.copy()
    sm.g2p_advect(state, sm.SimParams())
    assert np.abs(state.C - a).max() < 1e-4 * max(np.abs(a).max(), 1.0)
    assert np.abs(state.v - x_before @ a.T).max() < 1e-6 * max(np.abs(a).max(), 1.0)


def test_g2p_zero_velocities_keep_positions(small_grid, rng):
    """test_transfers.py:116-121: positions bit-identical (the device keeps
    fp32, and the host mirror keeps the caller's fp64 value wherever the
    device value is its fp32 rounding)."""
    state, _ = random_state(small_grid, 30, rng)
    state.grid_mv[:] = 0.0
    x0 = state.x.copy()
    sm.g2p_advect(state, sm.SimParams())
    assert np.array_equal(state.x, x0)


# ----------------------------------------------------------------- substeps
def make_block(grid, count=256, center=(0.5, 0.6, 0.5), size=(0.2, 0.2, 0.2), young=5.0e3):
    mats = [sm.Material(young, 0.3, 1000.0)]
    spawn = sm.sample_box(center, size, count, seed=11, grid=grid)
    return sm.SimState.from_spawns(grid, [spawn], mats), mats


def test_free_fall_matches_ballistics(small_grid):
    """test_substep.py:15-24 (fp32 velocity accumulated over 100 substeps)."""
    state, mats = make_block(small_grid, count=1, center=(0.5, 0.7, 0.5), size=(0.01, 0.01, 0.01))
    params = sm.SimParams(gravity=(0.0, -9.8, 0.0))
    n = 100
    for _ in range(n):
        sm.substep(state, mats, params)
    expected = np.array([0.0, -9.8 * n * params.dt, 0.0])
    assert np.abs(state.v[0] - expected).max() < 1e-5
    assert state.time == pytest.approx(n * params.dt, rel=1e-12)


def test_rest_block_stays_put(small_grid):
    """test_substep.py:27-33."""
    state, mats = make_block(small_grid)
    params = sm.SimParams(gravity=(0.0, 0.0, 0.0))
    x0 = state.x.astype(np.float32).astype(np.float64)
    for _ in range(100):
        sm.substep(state, mats, params)
    assert np.abs(state.x - x0).max() < 1e-7


def test_block_on_floor_stays_stable():
    """test_substep.py:36-45 (1000 substeps through step())."""
    grid = sm.Grid(resolution=(32, 32, 32), extent=(1.0, 1.0, 1.0))
    state, mats = make_block(grid, count=1000, center=(0.5, 0.25, 0.5), size=(0.25, 0.25, 0.25))
    params = sm.SimParams()
    for _ in range(40):
        sm.step(state, mats, params)
    assert not state.has_nan()
    assert (state.x >= 0.0).all()
    assert (state.x <= np.array(grid.extent)).all()


def test_step_advances_sim_time(small_grid):
    """test_substep.py:48-55."""
    state, mats = make_block(small_grid)
    report = sm.step(state, mats, sm.SimParams())
    assert state.time == pytest.approx(0.0125, rel=1e-12)
    assert report.timings_ms["soft_simulation"] > 0.0
    assert "collision_detection" in report.timings_ms
    assert report.step_index == 1


def test_runs_are_bitwise_deterministic(small_grid):
    """test_substep.py:58-66: deterministic mode (fixed-order node gather)."""
    results = []
    for _ in range(2):
        state, mats = make_block(small_grid, count=300)
        params = sm.SimParams(deterministic=True)
        for _ in range(30):
            sm.substep(state, mats, params)
        results.append(state.x.copy())
    assert np.array_equal(results[0], results[1])


# ---------------------------------------------------------------- collision
def test_no_colliders_all_sentinel(small_grid):
    """test_collision.py:195-198."""
    field = sm.update_collision_field([], small_grid)
    assert (field.object_id == -1).all()
    assert (field.distance >= 1e29).all()


def test_merged_field_tie_goes_to_lowest(small_grid):
    """test_collision.py:218-225."""
    shape = sm.Box(np.array([0.1, 0.1, 0.1]))
    a = sm.RigidCollider(id=2, shape=shape, translation=np.array([0.4, 0.5, 0.5]))
    b = sm.RigidCollider(id=5, shape=shape, translation=np.array([0.4, 0.5, 0.5]))
    field = sm.update_collision_field([a, b], small_grid)
    hit = field.object_id >= 0
    assert hit.any()
    assert (field.object_id[hit] == 0).all()


def scalar_box_distance(c, px, py, pz):
    """test_collision.py:160-172: plain-arithmetic box distance in the
    collider frame (the kernel's operation order)."""
    d0, d1, d2 = px - c.translation[0], py - c.translation[1], pz - c.translation[2]
    r = c.rotation
    lx = r[0, 0] * d0 + r[1, 0] * d1 + r[2, 0] * d2
    ly = r[0, 1] * d0 + r[1, 1] * d1 + r[2, 1] * d2
    lz = r[0, 2] * d0 + r[1, 2] * d1 + r[2, 2] * d2
    h = c.shape.half_extents
    qx, qy, qz = abs(lx) - h[0], abs(ly) - h[1], abs(lz) - h[2]
    ox, oy, oz = max(qx, 0.0), max(qy, 0.0), max(qz, 0.0)
    return np.sqrt(ox * ox + oy * oy + oz * oz) + min(max(qx, qy, qz), 0.0)


def test_merged_field_matches_brute_force(rng):
    """test_collision.py:175-215: the merged field equals an independent
    per-node min/argmin loop, bit for bit."""
    grid = sm.Grid(resolution=(8, 8, 8), extent=(1.0, 1.0, 1.0))
    for _ in range(5):
        k = int(rng.integers(1, 5))
        colliders = [sm.RigidCollider(id=i, shape=sm.Box(rng.uniform(0.05, 0.3, 3)),
                                      rotation=Rotation.random(random_state=rng).as_matrix(),
                                      translation=rng.uniform(0.1, 0.9, 3)) for i in range(k)]
        theta = 0.5 * grid.dx
        field = sm.update_collision_field(colliders, grid, theta)
        dist = np.full(grid.resolution, 1e30)
        obj = np.full(grid.resolution, -1, dtype=np.int32)
        for ix, iy, iz in np.ndindex(*grid.resolution):
            best, bi = 1e30, -1
            for i, c in enumerate(colliders):
                d = scalar_box_distance(c, ix * grid.dx, iy * grid.dx, iz * grid.dx)
                if d < best:
                    best, bi = d, i
            dist[ix, iy, iz] = best
            obj[ix, iy, iz] = bi if best < 2.0 * theta else -1
        assert np.array_equal(field.object_id, obj)
        assert np.array_equal(field.distance, dist)


def test_grid_update_resolves_against_collider(small_grid):
    """test_collision.py:265-282: a falling block stops on a sticky tool."""
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.62, 0.5), (0.1, 0.1, 0.1), 64, seed=5, grid=small_grid)
    state = sm.SimState.from_spawns(small_grid, [spawn], mats)
    state.v[:, 1] = -1.0
    collider = sm.RigidCollider(id=0, shape=sm.Box(np.array([0.2, 0.05, 0.2])),
                                translation=np.array([0.5, 0.45, 0.5]), mode="sticky")
    params = sm.SimParams(gravity=(0.0, 0.0, 0.0))
    for _ in range(40):
        sm.substep(state, mats, params, [collider])
    assert state.x[:, 1].min() > 0.45 + 0.05 - 2.5 * small_grid.dx
