"""Batched independent environments (BASELINE config 4: RL rollouts).

E environments with identical grids are packed as tiles of ONE device
context: tile e occupies nodes [o_e, o_e + res) of a grid of
tiles[0] x tiles[1] x tiles[2] environment tiles.  The kernels keep every
environment's particles inside its own tile margins (core.py:51-56 applied per
tile) and apply domain walls and colliders per tile (include/softmpm_b200.h:
env_tiles / colliders_per_env), so environments never interact while one
launch sweeps all of them -- small scenes stop being launch/latency bound.

Across GPUs, environments are sharded contiguously by rank (``shard``); the
stepping needs no collective (``step`` is independent per rank).

Semantics per environment are those of ``core.step`` on that environment
alone: pose_fn(colliders_e, t) before every substep, F7 frozen collider modes
(SimParams.collider_mode="live" to opt out), ``time += dt`` per substep.
Results match an isolated run up to fp32 rounding of the shifted positions.
"""

from __future__ import annotations

import math
import time as _time

import numpy as np

from . import core
from .collision import RigidCollider
from .errors import ParameterError


def shard(n_envs: int, world: int, rank: int) -> range:
    """Contiguous block of environment indices owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_envs, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def tile_shape(n: int) -> tuple[int, int, int]:
    """Near-cubic (tx, ty, tz) with tx * ty * tz >= n (few empty tiles)."""
    best = None
    for tx in range(1, n + 1):
        for ty in range(1, n // tx + 2):
            tz = math.ceil(n / (tx * ty))
            cand = (tx, ty, tz)
            waste = tx * ty * tz - n
            key = (waste, max(cand) - min(cand))
            if best is None or key < best[0]:
                best = (key, cand)
        if tx * tx * tx > 4 * n:
            break
    return best[1]


class EnvBatch:
    """E independent scenes stepped together on one GPU."""

    def __init__(self, states: list, colliders: list[list[RigidCollider]] | None = None,
                 tiles: tuple[int, int, int] | None = None, device: int | None = None):
        if not states:
            raise ParameterError("EnvBatch needs at least one environment")
        g0 = states[0].grid
        for st in states:
            if st.grid.resolution != g0.resolution or st.grid.extent != g0.extent:
                raise ParameterError("all environments must share one Grid")
        self.n_envs = len(states)
        self.tiles = tuple(tiles) if tiles else tile_shape(self.n_envs)
        if int(np.prod(self.tiles)) < self.n_envs:
            raise ParameterError(f"tiles {self.tiles} hold fewer than {self.n_envs} environments")
        self.env_grid = g0
        res = tuple(r * t for r, t in zip(g0.resolution, self.tiles))
        ext = tuple(e * t for e, t in zip(g0.extent, self.tiles))
        self.grid = core.Grid(res, ext)
        self.origins = np.array([self._origin(e) for e in range(self.n_envs)])
        counts = [st.particle_count for st in states]
        self.offsets = np.concatenate([[0], np.cumsum(counts)])
        cat = lambda f: np.concatenate([getattr(st, f) for st in states])
        x = np.concatenate([st.x + self.origins[e] for e, st in enumerate(states)])
        self.state = core.SimState(self.grid, x, cat("v"), cat("F"), cat("C"), cat("mass"),
                                   cat("vol0"), cat("material_id"), device=device)
        self.state._env_tiles = self.tiles
        self.colliders = colliders or [[] for _ in states]
        if len(self.colliders) != self.n_envs:
            raise ParameterError("one collider list per environment")
        k = {len(c) for c in self.colliders}
        if len(k) != 1:
            raise ParameterError("every environment needs the same number of colliders")
        self.k = k.pop()
        # device-side proxies in global coordinates (identity fixed -> F7 caching holds);
        # empty tiles (tiles > envs) get parked copies of environment 0's tools
        self._proxies = []
        n_tiles = int(np.prod(self.tiles))
        for e in range(n_tiles):
            src = self.colliders[min(e, self.n_envs - 1)]
            for c in src:
                self._proxies.append(RigidCollider(id=len(self._proxies), shape=c.shape,
                                                   friction_mu=c.friction_mu, mode=c.mode))
        self.state._colliders_per_env = self.k if self.k else 0
        self.time = 0.0
        self.step_count = 0

    def _origin(self, e: int) -> np.ndarray:
        tx, ty, tz = self.tiles
        i, rem = divmod(e, ty * tz)
        j, kk = divmod(rem, tz)
        return np.array([i, j, kk], dtype=np.float64) * np.array(self.env_grid.extent)

    def _sync_proxies(self, e: int) -> None:
        o = self.origins[e]
        for ci, c in enumerate(self.colliders[e]):
            px = self._proxies[e * self.k + ci]
            px.set_pose(c.rotation, c.translation + o, c.linear_velocity, c.angular_velocity)
            px.mode = c.mode

    def _tile_proxies_park(self) -> None:
        n_tiles = int(np.prod(self.tiles))
        for t in range(self.n_envs, n_tiles):
            o = self._origin_tile(t)
            for ci in range(self.k):
                src = self.colliders[self.n_envs - 1][ci]
                px = self._proxies[t * self.k + ci]
                px.set_pose(src.rotation, src.translation + o, np.zeros(3), np.zeros(3))

    def _origin_tile(self, t: int) -> np.ndarray:
        tx, ty, tz = self.tiles
        i, rem = divmod(t, ty * tz)
        j, kk = divmod(rem, tz)
        return np.array([i, j, kk], dtype=np.float64) * np.array(self.env_grid.extent)

    def pose_rows(self, poses: dict) -> tuple:
        """Pose table from per-environment arrays in environment-local frames.

        poses: {"R": (nsub, E, k, 3, 3), "T": (nsub, E, k, 3), "lv": ..., "av": ...}
        (the vectorised feed an RL policy produces); modes stay frozen/packed.
        """
        nsub = poses["T"].shape[0]
        n_tiles = int(np.prod(self.tiles))
        R = np.empty((nsub, n_tiles, self.k, 3, 3))
        T = np.empty((nsub, n_tiles, self.k, 3))
        lv = np.zeros((nsub, n_tiles, self.k, 3))
        av = np.zeros((nsub, n_tiles, self.k, 3))
        E = self.n_envs
        R[:, :E] = poses["R"]
        T[:, :E] = poses["T"] + self.origins[None, :, None, :]
        lv[:, :E] = poses.get("lv", 0.0)
        av[:, :E] = poses.get("av", 0.0)
        if n_tiles > E:  # parked tools of empty tiles
            park = np.array([self._origin_tile(t) for t in range(E, n_tiles)])
            R[:, E:] = poses["R"][:, -1:]
            T[:, E:] = poses["T"][:, -1:] + park[None, :, None, :]
        pk = self.state._packed_colliders(self._proxies)
        md = np.broadcast_to(pk.mode, (nsub, len(pk.mode)))
        flat = lambda a, *tail: np.ascontiguousarray(a.reshape((nsub, n_tiles * self.k) + tail))
        return (flat(R, 3, 3), flat(T, 3), flat(lv, 3), flat(av, 3), np.ascontiguousarray(md, np.int32))

    def step(self, materials, params: core.SimParams, pose_fns=None, poses: dict | None = None) -> core.StepReport:
        """One frame of params.substeps_per_frame substeps for every environment.

        Tool kinematics come either from per-environment ``pose_fns`` (the
        reference's pose_fn(colliders, t) protocol) or from a vectorised
        ``poses`` table (see pose_rows)."""
        st = self.state
        nsub = params.substeps_per_frame
        t_col = 0.0
        rows = None
        if self.k and poses is not None:
            t0 = _time.perf_counter()
            rows = self.pose_rows(poses)
            t_col = _time.perf_counter() - t0
        elif self.k:
            t0 = _time.perf_counter()
            R, T, lv, av, md = [], [], [], [], []
            t = self.time
            for _ in range(nsub):
                for e in range(self.n_envs):
                    if pose_fns is not None and pose_fns[e] is not None:
                        pose_fns[e](self.colliders[e], t)
                    self._sync_proxies(e)
                self._tile_proxies_park()
                pk = st._packed_colliders(self._proxies, params)
                R.append(pk.rotation.copy())
                T.append(pk.translation.copy())
                lv.append(pk.linear_velocity.copy())
                av.append(pk.angular_velocity.copy())
                md.append(pk.mode.copy())
                t += params.dt
            rows = (np.ascontiguousarray(R), np.ascontiguousarray(T), np.ascontiguousarray(lv),
                    np.ascontiguousarray(av), np.ascontiguousarray(md, np.int32))
            t_col = _time.perf_counter() - t0
        t0 = _time.perf_counter()
        inv, _ = core._run_substeps(st, materials, params, self._proxies if self.k else [], nsub, rows)
        t_soft = _time.perf_counter() - t0
        for _ in range(nsub):
            self.time += params.dt
        st.time = self.time
        self.step_count += 1
        return core.StepReport(step_index=self.step_count, sim_time=self.time,
                               timings_ms={"collision_detection": 1000.0 * t_col,
                                           "soft_simulation": 1000.0 * t_soft},
                               inverted_particles=inv)

    # ---- per-environment readback (environment-local coordinates) --------
    def env_slice(self, e: int) -> slice:
        return slice(int(self.offsets[e]), int(self.offsets[e + 1]))

    def x(self, e: int) -> np.ndarray:
        return self.state.x[self.env_slice(e)] - self.origins[e]

    def field(self, name: str, e: int) -> np.ndarray:
        if name == "x":
            return self.x(e)
        return getattr(self.state, name)[self.env_slice(e)]

    @property
    def particle_count(self) -> int:
        return self.state.particle_count
