"""Tool-kinematics input: keyframe trajectories -> per-substep collider poses.

Restates the reference's kinematics feed (/root/reference/pkg/src/softmpm/
scene.py:143-183 ``pose_at``, 286-305 ``_apply_poses`` / ``make_pose_fn``):
positions interpolate linearly, orientations spherically (scipy Rotation),
velocities are segment-constant, out-of-range times clamp with zero velocity,
and closing a gripper group's jaws switches its members to sticky contact
(which ``step`` then ignores in F7-compat mode, exactly like the reference).

``pose_fn(colliders, t)`` is the only thing ``core.step`` needs; a PyBullet
adapter would simply call ``RigidCollider.set_pose`` from
``getBasePositionAndOrientation`` / ``getBaseVelocity`` inside one.  The
reference's JSON scene schema and builtin scenario library are out of scope
(host-side setup).
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


def make_pose_fn(trajectory: list[Keyframe], groups: list[GripperGroup] | None = None,
                 base_mode: dict | None = None):
    """Kinematics feed for ``step``: sets collider poses at substep times."""
    if not trajectory:
        return None

    def pose_fn(colliders, t):
        poses, jaw = pose_at(trajectory, t)
        apply_poses(colliders, poses, jaw, groups, base_mode)

    return pose_fn
