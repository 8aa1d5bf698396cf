"""Tool-kinematics input: keyframe trajectories -> per-substep collider poses.

Restates the reference's kinematics feed (/root/reference/pkg/src/softmpm/
scene.py:143-183 ``pose_at``, 286-305 ``_apply_poses`` / ``make_pose_fn``):
positions interpolate linearly, orientations spherically (scipy Rotation),
velocities are segment-constant, out-of-range times clamp with zero velocity,
and closing a gripper group's jaws switches its members to sticky contact
(which ``step`` then ignores in F7-compat mode, exactly like the reference).

``pose_fn(colliders, t)`` is the only thing ``core.step`` needs;
``pybullet_pose_fn`` is one over a PyBullet simulation (the tools follow
rigid bodies: ``getBasePositionAndOrientation`` / ``getBaseVelocity`` ->
``RigidCollider.set_pose``, collision.py:74-82).  The reference's JSON scene
schema and builtin scenario library are out of scope (host-side setup).
"""

from __future__ import annotations

from bisect import bisect_right
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial.transform import Rotation

from .errors import SceneError


@dataclass
class Keyframe:
    time: float
    poses: list  # per collider: (T (3,), quaternion xyzw (4,))
    jaw_state: str = "open"


@dataclass
class GripperGroup:
    name: str
    colliders: list[int]
    jaw_axis: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0]))
    open_gap: float = 0.1
    closed_gap: float = 0.02


def _normalized(q) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    return q / np.linalg.norm(q)


def pose_at(trajectory: list[Keyframe], t: float):
    """(poses, jaw_state); poses[i] = (T, R 3x3, linear_velocity, angular_velocity)."""
    if not trajectory:
        raise SceneError("empty trajectory")
    zero = np.zeros(3)

    def fixed(kf: Keyframe):
        return [(np.asarray(T, dtype=np.float64), Rotation.from_quat(_normalized(q)).as_matrix(),
                 zero, zero) for T, q in kf.poses], kf.jaw_state

    times = [k.time for k in trajectory]
    if t <= times[0]:
        return fixed(trajectory[0])
    if t >= times[-1]:
        return fixed(trajectory[-1])
    i = bisect_right(times, t) - 1
    a, b = trajectory[i], trajectory[i + 1]
    seg = b.time - a.time
    s = (t - a.time) / seg
    out = []
    for (ta, qa), (tb, qb) in zip(a.poses, b.poses):
        ta = np.asarray(ta, dtype=np.float64)
        tb = np.asarray(tb, dtype=np.float64)
        ra = Rotation.from_quat(_normalized(qa))
        rb = Rotation.from_quat(_normalized(qb))
        rel = (ra.inv() * rb).as_rotvec()
        rot = (ra * Rotation.from_rotvec(rel * s)).as_matrix()
        out.append(((1.0 - s) * ta + s * tb, rot, (tb - ta) / seg, ra.apply(rel) / seg))
    return out, a.jaw_state


def apply_poses(colliders, poses, jaw: str, groups: list[GripperGroup] | None = None,
                base_mode: dict | None = None) -> None:
    grouped = {cid for g in (groups or []) for cid in g.colliders}
    for col, (T, R, lv, av) in zip(colliders, poses):
        col.set_pose(R, T, lv, av)
        if col.id in grouped:
            col.mode = "sticky" if jaw == "closed" else (base_mode or {}).get(col.id, "coulomb")


def _rotvec_matrix(rv: np.ndarray) -> np.ndarray:
    """Rotation matrices of rotation vectors (..., 3) (Rodrigues)."""
    rv = np.asarray(rv, dtype=np.float64)
    th = np.linalg.norm(rv, axis=-1)
    safe = np.where(th > 0.0, th, 1.0)
    k = rv / safe[..., None]
    K = np.zeros(rv.shape[:-1] + (3, 3))
    K[..., 0, 1], K[..., 0, 2] = -k[..., 2], k[..., 1]
    K[..., 1, 0], K[..., 1, 2] = k[..., 2], -k[..., 0]
    K[..., 2, 0], K[..., 2, 1] = -k[..., 1], k[..., 0]
    s, c = np.sin(th)[..., None, None], (1.0 - np.cos(th))[..., None, None]
    R = np.eye(3) + s * K + c * (K @ K)
    return np.where((th > 0.0)[..., None, None], R, np.eye(3))


class _CompiledTrajectory:
    """pose_at with the per-keyframe / per-segment scipy work done once: a
    substep pose is a lerp plus R_a exp(s rel) (Rodrigues; equal to scipy's
    quaternion slerp to ~1e-16).  ``table(times)`` evaluates many substeps in
    one vectorised pass -- the per-frame pose table core.step uploads."""

    def __init__(self, trajectory: list[Keyframe]):
        self.times = np.array([k.time for k in trajectory], dtype=np.float64)
        self.jaw = [k.jaw_state for k in trajectory]
        self.T = np.array([[np.asarray(T, dtype=np.float64) for T, _ in k.poses] for k in trajectory])
        rots = [[Rotation.from_quat(_normalized(q)) for _, q in k.poses] for k in trajectory]
        self.R = np.array([[r.as_matrix() for r in row] for row in rots])
        nk = len(trajectory)
        ncol = self.T.shape[1]
        self.rel = np.zeros((max(nk - 1, 0), ncol, 3))
        self.av = np.zeros((max(nk - 1, 0), ncol, 3))
        for i in range(nk - 1):
            seg = self.times[i + 1] - self.times[i]
            for c in range(ncol):
                ra, rb = rots[i][c], rots[i + 1][c]
                rel = (ra.inv() * rb).as_rotvec()
                self.rel[i, c] = rel
                self.av[i, c] = ra.apply(rel) / seg

    def table(self, times):
        """(R (n, k, 3, 3), T (n, k, 3), lv, av, jaw states) at `times`."""
        t = np.asarray(times, dtype=np.float64)
        nk = len(self.times)
        clamp_lo, clamp_hi = t <= self.times[0], t >= self.times[-1]
        if nk < 2:
            n = len(t)
            return (np.broadcast_to(self.R[0], (n,) + self.R[0].shape).copy(),
                    np.broadcast_to(self.T[0], (n,) + self.T[0].shape).copy(),
                    np.zeros((n,) + self.T[0].shape), np.zeros((n,) + self.T[0].shape), [self.jaw[0]] * n)
        a = np.clip(np.searchsorted(self.times, t, side="right") - 1, 0, nk - 2)
        seg = self.times[a + 1] - self.times[a]
        s = ((t - self.times[a]) / seg)[:, None, None]
        T = (1.0 - s) * self.T[a] + s * self.T[a + 1]
        R = self.R[a] @ _rotvec_matrix(self.rel[a] * s)
        lv = (self.T[a + 1] - self.T[a]) / seg[:, None, None]
        av = self.av[a].copy()
        for mask, k in ((clamp_lo, 0), (clamp_hi, nk - 1)):
            if mask.any():
                R[mask], T[mask], lv[mask], av[mask] = self.R[k], self.T[k], 0.0, 0.0
        jaw = [self.jaw[0] if clamp_lo[j] else self.jaw[-1] if clamp_hi[j] else self.jaw[a[j]] for j in range(len(t))]
        return R, T, lv, av, jaw


class PoseFn:
    """``make_pose_fn``'s kinematics feed: ``pose_fn(colliders, t)`` sets the
    collider poses at time t (scene.py:286-305); ``core.step`` asks it for a
    whole frame's pose table at once (``table``)."""

    def __init__(self, trajectory, groups=None, base_mode=None):
        self.trajectory = trajectory
        self.groups = groups
        self.base_mode = base_mode
        self._compiled = _CompiledTrajectory(trajectory)

    def __call__(self, colliders, t):
        R, T, lv, av, jaw = self._compiled.table([t])
        poses = [(T[0, c], R[0, c], lv[0, c], av[0, c]) for c in range(T.shape[1])]
        apply_poses(colliders, poses, jaw[0], self.groups, self.base_mode)

    def table(self, colliders, times):
        """Per-substep (R, T, lv, av) arrays and the colliders' modes after
        each pose update (jaw-driven for gripper groups); leaves the colliders
        at the last time, as the per-substep calls would."""
        R, T, lv, av, jaw = self._compiled.table(times)
        grouped = {cid for g in (self.groups or []) for cid in g.colliders}
        modes = []
        for j in range(len(times)):
            row = []
            for c in colliders:
                if c.id in grouped:
                    row.append("sticky" if jaw[j] == "closed" else (self.base_mode or {}).get(c.id, "coulomb"))
                else:
                    row.append(c.mode)
            modes.append(row)
        last = len(times) - 1
        self.__call__(colliders, times[last]) if last >= 0 else None
        return R, T, lv, av, modes


def make_pose_fn(trajectory: list[Keyframe], groups: list[GripperGroup] | None = None,
                 base_mode: dict | None = None):
    """Kinematics feed for ``step``: sets collider poses at substep times."""
    if not trajectory:
        return None
    return PoseFn(trajectory, groups, base_mode)


def pybullet_pose_fn(pb, body_ids, client=None):
    """A ``pose_fn`` whose collider k follows PyBullet body ``body_ids[k]``:
    base position / orientation (xyzw quaternion) give T and R, base linear /
    angular velocity give the contact's rigid-motion velocity (kernels.py:
    377-383).  ``pb`` is the ``pybullet`` module (or anything with its two
    functions); PyBullet owns the clock, so the substep time is not used --
    step the rigid-body world between frames, or every substep from a
    pose_fn that wraps this one.  Each call reads every body once."""
    kw = {} if client is None else {"physicsClientId": client}

    def pose_fn(colliders, t):
        for c, b in zip(colliders, body_ids):
            pos, orn = pb.getBasePositionAndOrientation(b, **kw)
            lin, ang = pb.getBaseVelocity(b, **kw)
            c.set_pose(Rotation.from_quat(np.asarray(orn, dtype=np.float64)).as_matrix(),
                       np.asarray(pos, dtype=np.float64), lin, ang)

    return pose_fn

