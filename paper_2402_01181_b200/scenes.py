"""Synthetic tissue scenes of BASELINE.json's configs.

Defaults follow the reference scenarios (scenarios.py:62-64: E = 1e4 Pa,
nu = 0.3, rho = 1000) and SimParams (dt 5e-4, 25 substeps, clamp boundary
width 3, theta = 0.5 dx).  Each builder returns (state, materials, params,
colliders, pose_fn).

  c1  30 K block dropped into the floor band, 64^3, no tools
  c2  30 K block, 128^3, two baked-SDF capsule jaws (grasper) on a
      down -> close -> pull keyframe path, Coulomb mu = 0.35 (sticky when closed)
  c3  1 M slab on 256^3 pressed 3 cm deep by a box tool moving down at 0.5 m/s,
      then held (a deeper press at this dt exceeds the explicit CFL limit at
      256^3 -- the CPU oracle and the GPU path blow up alike)
"""

from __future__ import annotations

import numpy as np

from .collision import Baked, Box, RigidCollider
from .core import Grid, SimParams, SimState
from .materials import Material
from .sampling import sample_box
from .scene import GripperGroup, Keyframe, make_pose_fn
from .sdf import bake_capsule

_Q = np.array([0.0, 0.0, 0.0, 1.0])


def _material():
    return [Material(1.0e4, 0.3, 1000.0)]


def c1(count: int = 30_000, res: int = 64, seed: int = 1):
    grid = Grid((res, res, res))
    mats = _material()
    spawn = sample_box((0.5, 0.13, 0.5), (0.3, 0.2, 0.3), count, seed=seed, grid=grid)
    st = SimState.from_spawns(grid, [spawn], mats)
    return st, mats, SimParams(), [], None


def c2(count: int = 30_000, res: int = 128, seed: int = 1, sdf_res: int = 64):
    grid = Grid((res, res, res))
    mats = _material()
    spawn = sample_box((0.5, 0.13, 0.5), (0.3, 0.2, 0.3), count, seed=seed, grid=grid)
    st = SimState.from_spawns(grid, [spawn], mats)
    jaw = bake_capsule(radius=0.02, half_length=0.06, resolution=sdf_res, axis=1)
    cols = [RigidCollider(id=0, shape=Baked(jaw), friction_mu=0.35),
            RigidCollider(id=1, shape=Baked(jaw), friction_mu=0.35)]
    half_gap_open, half_gap_closed = 0.07, 0.035
    waypoints = [(0.0, (0.5, 0.40, 0.5), "open"), (0.25, (0.5, 0.26, 0.5), "open"),
                 (0.35, (0.5, 0.26, 0.5), "closed"), (0.8, (0.5, 0.42, 0.5), "closed")]
    traj = []
    for t, c, jawstate in waypoints:
        g = half_gap_closed if jawstate == "closed" else half_gap_open
        c = np.asarray(c)
        traj.append(Keyframe(t, [(c - [g, 0, 0], _Q), (c + [g, 0, 0], _Q)], jawstate))
    pose_fn = make_pose_fn(traj, [GripperGroup("grasper", [0, 1])], {0: "coulomb", 1: "coulomb"})
    pose_fn(cols, 0.0)
    return st, mats, SimParams(), cols, pose_fn


def c3(count: int = 1_000_000, res: int = 256, seed: int = 1):
    grid = Grid((res, res, res))
    mats = _material()
    spawn = sample_box((0.5, 0.1, 0.5), (0.5, 0.0977, 0.5), count, seed=seed, grid=grid)
    st = SimState.from_spawns(grid, [spawn], mats)
    top = 0.1 + 0.5 * 0.0977
    half = np.array([0.08, 0.03, 0.08])
    y0 = top + half[1] + 0.005
    press = 0.035  # 0.5 cm gap + 3 cm into the tissue
    traj = [Keyframe(0.0, [(np.array([0.5, y0, 0.5]), _Q)]),
            Keyframe(press / 0.5, [(np.array([0.5, y0 - press, 0.5]), _Q)]),
            Keyframe(10.0, [(np.array([0.5, y0 - press, 0.5]), _Q)])]
    cols = [RigidCollider(id=0, shape=Box(half), friction_mu=0.4)]
    pose_fn = make_pose_fn(traj)
    pose_fn(cols, 0.0)
    return st, mats, SimParams(), cols, pose_fn


def c4_trajectory():
    """Tool path of every config-4 environment: press 2.5 cm at 0.5 m/s, hold."""
    y0 = 0.23 + 0.035 + 0.005
    return [Keyframe(0.0, [(np.array([0.5, y0, 0.5]), _Q)]),
            Keyframe(0.05, [(np.array([0.5, y0 - 0.025, 0.5]), _Q)]),
            Keyframe(10.0, [(np.array([0.5, y0 - 0.025, 0.5]), _Q)])]


def c4_envs(n_envs: int = 1024, count: int = 30_000, res: int = 64, first_seed: int = 1,
            env_ids=None):
    """Config 4: independent config-1-style environments (seed = env index),
    each with a box tool pressing 2 cm into its block at 0.5 m/s then holding;
    returns an EnvBatch plus (materials, params, pose_fns)."""
    from .batch import EnvBatch

    ids = list(env_ids) if env_ids is not None else list(range(n_envs))
    grid = Grid((res, res, res))
    mats = _material()
    states, cols, fns = [], [], []
    for e in ids:
        spawn = sample_box((0.5, 0.13, 0.5), (0.3, 0.2, 0.3), count, seed=first_seed + e, grid=grid)
        states.append(SimState.from_spawns(grid, [spawn], mats))
        traj = c4_trajectory()
        c = [RigidCollider(id=0, shape=Box(np.array([0.06, 0.035, 0.06])), friction_mu=0.4)]
        fn = make_pose_fn(traj)
        fn(c, 0.0)
        cols.append(c)
        fns.append(fn)
    return EnvBatch(states, cols), mats, SimParams(), fns


def c5_spawn(count: int = 64_000_000, res: int = 1024, seed: int = 1):
    """Config 5's grid, particle spawn, materials and params without the
    SimState (slab ranks build only their own window: slab.rank_window)."""
    grid = Grid((res, res, res))
    spawn = sample_box((0.5, 0.065, 0.5), (0.4, 0.1, 0.4), count, seed=seed, grid=grid)
    return grid, spawn, _material(), SimParams(dt=1.0e-4, rebin_interval=5)


def c5(count: int = 64_000_000, res: int = 1024, seed: int = 1):
    """Config 5: a large tissue volume (0.4 x 0.1 x 0.4 m, ~3.7 particles per
    cell at 1024^3) settling on the floor under gravity; slab-decomposed along x
    across ranks by slab.split_state / bench.py --config c5.  dt = 1e-4: at
    dx ~ 1 mm the default 5e-4 breaks the explicit CFL bound (elastic wave
    speed ~3.7 m/s -> c dt / dx ~ 1.9), for the reference scheme as well."""
    grid, spawn, mats, params = c5_spawn(count, res, seed)
    st = SimState.from_spawns(grid, [spawn], mats)
    return st, mats, params, [], None


BUILDERS = {"c1": c1, "c2": c2, "c3": c3, "c5": c5}
