"""GPU scene-level parity: BASELINE configs (scaled) against the CPU oracle O1
fed the same per-substep tool poses, plus the install() re-routing of a
reference-shaped module."""
import types
from dataclasses import dataclass, field

import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import scenes
from conftest import load_golden, rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle_for(st, mats, theta=True):
    g = st.grid
    return O.OracleSim(O.OracleParams(res=g.resolution, dx=g.dx, theta=0.5 * g.dx if theta else -1.0),
                       st.x, st.v, st.F, st.C, st.mass, st.vol0, st.material_id, mats[0].mu,
                       mats[0].lam)


def _run_pair(st, mats, params, cols, ocols, pose_fn, frames, live=False):
    osim = _oracle_for(st, mats)
    packed = None
    t = 0.0
    for _ in range(frames):
        sm.step(st, mats, params, cols, pose_fn)
        for _ in range(params.substeps_per_frame):
            pose_fn(ocols, t)
            if packed is None or live:
                packed = sm.pack_colliders(ocols)   # live: modes re-read every substep
            else:
                packed.refresh_poses(ocols)         # frozen (reference F7)
            osim.substep(packed)
            t += params.dt
    return osim


@pytest.mark.parametrize("live", [False, True])
def test_c2_capsule_grasper_matches_oracle(live):
    """Config 2 (scaled): baked-SDF capsule jaws go down, close (sticky) and pull."""
    st, mats, params, cols, pose_fn = scenes.c2(count=8000, res=64, sdf_res=32)
    _, _, _, ocols, _ = scenes.c2(count=8000, res=64, sdf_res=32)
    params = sm.SimParams(collider_mode="live" if live else "frozen")
    osim = _run_pair(st, mats, params, cols, ocols, pose_fn, frames=36, live=live)  # jaws close at t=0.35
    assert st.time == pytest.approx(osim.time, rel=1e-12)
    assert (st._collision.object_id >= 0).sum() > 0
    for k in ("x", "v", "F"):
        assert rel_l2(getattr(st, k), getattr(osim, k)) < 1e-3, k
    if live:
        assert [c.mode for c in cols] == ["sticky", "sticky"]


def test_c3_press_scaled_matches_oracle():
    """Config 3 (scaled to 64^3): box press and hold."""
    st, mats, params, cols, pose_fn = scenes.c3(count=60000, res=64)
    _, _, _, ocols, _ = scenes.c3(count=60000, res=64)
    osim = _run_pair(st, mats, params, cols, ocols, pose_fn, frames=8)
    for k in ("x", "v", "F"):
        assert rel_l2(getattr(st, k), getattr(osim, k)) < 1e-3, k


@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_cross_frame_stretches_match_oracle(cfg, monkeypatch):
    """Option rebin_frames (SOFTMPM_REBIN_FRAMES=3): frames of an untouched
    state keep the particle order and work list of a re-binning up to two
    frames old (item bounds recomputed exactly at each frame's first
    substep; particles that drifted off their tiles take the float path)."""
    monkeypatch.setenv("SOFTMPM_REBIN_FRAMES", "3")
    if cfg == "c3":
        st, mats, params, cols, pose_fn = scenes.c3(count=60000, res=64)
        _, _, _, ocols, _ = scenes.c3(count=60000, res=64)
        osim = _run_pair(st, mats, params, cols, ocols, pose_fn, frames=8)
        tol = 1e-3
    else:
        st, mats, params, _, _ = scenes.c1(count=30000, res=64)
        osim = _oracle_for(st, mats, theta=False)
        per_frame = []
        for _ in range(6):
            l0 = st._ctx.launches if st._ctx is not None else 0
            sm.step(st, mats, params)
            per_frame.append(st._ctx.launches - l0)
            for _ in range(params.substeps_per_frame):
                osim.substep(None)
        assert min(per_frame[1:]) < max(per_frame[1:]), per_frame  # some frames kept their bins
        tol = 1e-4
    for k in ("x", "v", "F"):
        assert rel_l2(getattr(st, k), getattr(osim, k)) < tol, k


def test_c1_floor_drop_matches_oracle_and_rebin_interval():
    st, mats, params, _, _ = scenes.c1(count=30000, res=64)
    osim = _oracle_for(st, mats, theta=False)
    for interval in (25, 5):
        p = sm.SimParams(rebin_interval=interval)
        sm.step(st, mats, p)
        for _ in range(p.substeps_per_frame):
            osim.substep(None)
    for k in ("x", "v", "F"):
        assert rel_l2(getattr(st, k), getattr(osim, k)) < 1e-4, k


def _fake_softmpm():
    """A module shaped like the reference softmpm (core.SimState dataclass with
    numpy fields, StepReport, p2g/grid_update/g2p_advect/substep/step)."""
    core = types.ModuleType("softmpm.core")

    @dataclass
    class Grid:
        resolution: tuple
        extent: tuple = (1.0, 1.0, 1.0)

        @property
        def dx(self):
            return self.extent[0] / self.resolution[0]

    @dataclass
    class StepReport:
        step_index: int
        sim_time: float
        timings_ms: dict
        inverted_particles: int

    @dataclass
    class SimState:
        grid: Grid
        x: np.ndarray
        v: np.ndarray
        F: np.ndarray
        C: np.ndarray
        mass: np.ndarray
        vol0: np.ndarray
        material_id: np.ndarray
        time: float = 0.0
        step_count: int = 0
        grid_mv: np.ndarray = field(init=False)
        grid_m: np.ndarray = field(init=False)

        def __post_init__(self):
            self.grid_mv = np.zeros(tuple(self.grid.resolution) + (3,))
            self.grid_m = np.zeros(tuple(self.grid.resolution))

    def _ref_only(*a, **k):
        raise AssertionError("reference CPU path called after install()")

    core.Grid, core.StepReport, core.SimState = Grid, StepReport, SimState
    for nm in ("p2g", "grid_update", "g2p_advect", "substep", "step"):
        setattr(core, nm, _ref_only)
    mod = types.ModuleType("softmpm")
    mod.core = core
    for nm in ("p2g", "grid_update", "g2p_advect", "substep", "step"):
        setattr(mod, nm, _ref_only)
    return mod


def test_install_reroutes_reference_shaped_module():
    g = load_golden("floor_block.npz")
    ref = _fake_softmpm()
    sm.install(ref)
    try:
        res = tuple(int(r) for r in g["res"])
        st = ref.core.SimState(ref.core.Grid(res), g["in_x"].copy(), g["in_v"].copy(), g["in_F"].copy(),
                               g["in_C"].copy(), g["mass"], g["vol0"], np.zeros(len(g["in_x"]), np.int32))
        mats = [sm.Material(float(g["E"]), float(g["nu"]), float(g["rho"]))]
        x_obj = st.x
        inv = ref.substep(st, mats, sm.SimParams())
        assert inv == 0
        assert st.x is x_obj  # results land in the caller's arrays
        for k in ("x", "v", "F"):
            assert rel_l2(getattr(st, k), g[f"s1_{k}"]) < 1e-5, k
        assert st.grid_m.sum() == pytest.approx(g["mass"].sum(), rel=1e-5)
        rep = ref.step(st, mats, sm.SimParams(substeps_per_frame=9))
        assert isinstance(rep, ref.core.StepReport) and rep.step_index == 1
        for k in ("x", "v", "F"):
            assert rel_l2(getattr(st, k), g[f"s10_{k}"]) < 1e-4, k
    finally:
        sm.uninstall(ref)
    with pytest.raises(AssertionError):
        ref.step(st, mats, sm.SimParams())


def test_env_batch_matches_isolated_runs_and_oracle():
    """Config 4: environments packed as tiles of one context behave like
    isolated runs (and like the CPU oracle), with per-tile walls and tools."""
    ids = [0, 1, 2, 3, 4]
    batch, mats, params, fns = scenes.c4_envs(n_envs=5, count=4000, res=64, env_ids=ids)
    assert batch.tiles == (1, 1, 5) or int(np.prod(batch.tiles)) >= 5
    singles = [scenes.c4_envs(count=4000, res=64, env_ids=[e]) for e in ids]
    ref_b, _, _, ref_fns = scenes.c4_envs(count=4000, res=64, env_ids=[2])
    osim = _oracle_for(ref_b.state, mats)
    ocols = [sm.RigidCollider(id=0, shape=sm.Box(np.array([0.06, 0.035, 0.06])), friction_mu=0.4)]
    t = 0.0
    for _ in range(4):
        batch.step(mats, params, fns)
        for b1, _, _, f1 in singles:
            b1.step(mats, params, f1)
        for _ in range(params.substeps_per_frame):
            ref_fns[0](ocols, t)
            osim.substep(sm.pack_colliders(ocols))
            t += params.dt
    for e, (b1, _, _, _) in zip(ids, singles):
        for k in ("x", "v", "F"):
            assert rel_l2(batch.field(k, e), b1.field(k, 0)) < 1e-4, (e, k)
    for k in ("x", "v", "F"):
        assert rel_l2(batch.field(k, 2), getattr(osim, k)) < 1e-3, k
    # tools act: the pressed top layer moved down in every environment
    for e in ids:
        assert batch.field("v", e)[:, 1].min() < -0.05


def test_env_batch_vectorised_pose_table():
    batch, mats, params, fns = scenes.c4_envs(n_envs=3, count=3000, res=64)
    ref, _, _, rfns = scenes.c4_envs(n_envs=3, count=3000, res=64)
    nsub = params.substeps_per_frame
    t = np.arange(nsub) * params.dt
    R = np.broadcast_to(np.eye(3), (nsub, 3, 1, 3, 3)).copy()
    T = np.zeros((nsub, 3, 1, 3))
    lv = np.zeros((nsub, 3, 1, 3))
    for s in range(nsub):
        for e in range(3):
            poses, _ = sm.pose_at(_traj_c4(), t[s])
            T[s, e, 0] = poses[0][0]
            lv[s, e, 0] = poses[0][2]
    batch.step(mats, params, poses={"R": R, "T": T, "lv": lv})
    ref.step(mats, params, rfns)
    for e in range(3):
        assert rel_l2(batch.field("x", e), ref.field("x", e)) < 1e-6


def _traj_c4():
    q = np.array([0.0, 0.0, 0.0, 1.0])
    y0 = 0.23 + 0.035 + 0.005
    return [sm.Keyframe(0.0, [(np.array([0.5, y0, 0.5]), q)]),
            sm.Keyframe(0.05, [(np.array([0.5, y0 - 0.025, 0.5]), q)]),
            sm.Keyframe(10.0, [(np.array([0.5, y0 - 0.025, 0.5]), q)])]


def test_cooperative_substeps_kernel_matches_per_substep_launches():
    """Option "mega": substeps 2..L as one cooperative launch (fused phase,
    grid barrier, grid-op phase) reproduces the per-substep launches."""
    res = {}
    for mega in (0, 1):
        st, mats, params, cols, pose_fn = scenes.c2()
        params.rebin_interval = 10
        sm.step(st, mats, params, cols, pose_fn)  # creates the context
        st._ctx.call("mpm_set_option", b"mega", mega)
        for _ in range(4):
            sm.step(st, mats, params, cols, pose_fn)
        res[mega] = (st.x.copy(), st.v.copy(), st.F.copy())
    for a, b in zip(res[0], res[1]):
        assert rel_l2(a, b) < 1e-5


def test_programmatic_dependent_launch_matches_plain_launches():
    """Option "pdl": fused kernel and grid op launched with programmatic
    dependent launch (prologue overlapping the predecessor's tail) reproduce
    the plain stream-ordered launches on the tool-contact scene."""
    res = {}
    for pdl in (0, 1):
        st, mats, params, cols, pose_fn = scenes.c2()
        sm.step(st, mats, params, cols, pose_fn)
        st._ctx.call("mpm_set_option", b"pdl", pdl)
        for _ in range(4):
            sm.step(st, mats, params, cols, pose_fn)
        res[pdl] = (st.x.copy(), st.v.copy(), st.F.copy())
    for a, b in zip(res[0], res[1]):
        assert rel_l2(a, b) < 1e-5


def test_two_materials_match_oracle():
    """Per-particle material ids (SimParams materials list, materials.py:77-82):
    a stiff and a soft block side by side on the floor, 2 frames, against the
    O1 oracle with the same per-material (mu, lam)."""
    grid = sm.Grid((48, 48, 48))
    mats = [sm.Material(2.0e4, 0.3, 1000.0), sm.Material(3.0e3, 0.45, 1100.0)]
    a = sm.sample_box((0.35, 0.16, 0.5), (0.2, 0.15, 0.25), 6000, seed=1, grid=grid)
    b = sm.ParticleSpawn(sm.sample_box((0.65, 0.16, 0.5), (0.2, 0.15, 0.25), 6000, seed=2, grid=grid).positions,
                         a.rest_volume_per_particle, 1)
    st = sm.SimState.from_spawns(grid, [a, b], mats)
    assert set(np.unique(st.material_id)) == {0, 1}
    params = sm.SimParams()
    osim = O.OracleSim(O.OracleParams(res=grid.resolution, dx=grid.dx), st.x, st.v, st.F, st.C, st.mass, st.vol0,
                       st.material_id, [m.mu for m in mats], [m.lam for m in mats])
    for _ in range(2):
        sm.step(st, mats, params)
        for _ in range(params.substeps_per_frame):
            osim.substep(None)
    for k in ("x", "v", "F"):
        assert rel_l2(getattr(st, k), getattr(osim, k)) < 1e-4, k
