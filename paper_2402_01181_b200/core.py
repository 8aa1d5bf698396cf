"""Drop-in simulator API over the B200 kernels.

Same public surface and semantics as the reference's
/root/reference/pkg/src/softmpm/core.py -- ``Grid`` (24-56), ``SimParams``
(59-79), ``StepReport`` (82-89), ``SimState`` (92-169), ``bspline_weights``
(176-194), the stage operators ``p2g`` / ``grid_update`` / ``g2p_advect``
(211-258), ``substep`` (261-277) and ``step`` (280-320) -- but the state lives
on the GPU:

* ``SimState`` keeps x/v/F/C/mass/vol0 as fp32 SoA device buffers inside a
  C-ABI context (include/softmpm_b200.h) and exposes the reference's fp64
  numpy fields as lazily synchronised host mirrors: reading a field after a
  kernel downloads it (in place, so held references update), handing a field
  out or assigning it marks it for upload before the next kernel.
* ``step`` evaluates ``pose_fn`` for all substeps of the frame first (it
  depends only on t; the exact ``state.time += dt`` accumulation of
  core.py:315 is replayed) and uploads the resulting pose table once, so the
  whole frame runs device-resident.
* Collider ``mode`` changes are ignored after the first pack, exactly like
  the reference unless ``SimParams.collider_mode="live"``.

Extra ``SimParams`` fields (all defaulting to reference behaviour):
``stress_form`` ("kernel" = the reference kernel's F^-1 form, the drop-in
parity target; "spec" = materials.neo_hookean_stress's F^-T form),
``collider_mode`` ("frozen" | "live"), ``deterministic`` (sorted-order P2G
with bit-reproducible grid mass) and ``rebin_interval`` (substeps between
particle re-binning; the fast path's only tuning knob).
"""

from __future__ import annotations

import ctypes
import os
import time as _time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .collision import (MODE_NAMES, CollisionField, PackedColliders, RigidCollider,
                        pack_colliders)
from .errors import ParameterError, SpawnError, StencilError
from .materials import Material, pack_materials

_FIELDS = ("x", "v", "F", "C")
_FIELD_BIT = {"x": _lib.FIELD_X, "v": _lib.FIELD_V, "F": _lib.FIELD_F, "C": _lib.FIELD_C}
_KEEP_EQUAL = _lib.DOWNLOAD_KEEP_EQUAL


@dataclass(frozen=True)
class Grid:
    """Eulerian lattice: node i sits at i*dx per axis (core.py:24-56)."""

    resolution: tuple[int, int, int] = (64, 64, 64)
    extent: tuple[float, float, float] = (1.0, 1.0, 1.0)

    def __post_init__(self):
        object.__setattr__(self, "resolution", tuple(int(r) for r in self.resolution))
        object.__setattr__(self, "extent", tuple(float(e) for e in self.extent))
        if any(r < 8 for r in self.resolution):
            raise ParameterError(f"grid resolution too small: {self.resolution}")
        dxs = [e / r for e, r in zip(self.extent, self.resolution)]
        if max(dxs) - min(dxs) > 1.0e-12 * max(dxs):
            raise ParameterError(f"cell size must be uniform across axes, got {dxs}")
        if dxs[0] <= 0.0:
            raise ParameterError("grid extent must be positive")

    @property
    def dx(self) -> float:
        return self.extent[0] / self.resolution[0]

    @property
    def node_count(self) -> int:
        nx, ny, nz = self.resolution
        return nx * ny * nz

    def margin_bounds(self) -> tuple[np.ndarray, np.ndarray]:
        dx = self.dx
        lo = np.full(3, 1.5 * dx)
        hi = np.array([(r - 1.5 - 1.0e-7) * dx for r in self.resolution])
        return lo, hi


@dataclass
class SimParams:
    dt: float = 5.0e-4
    substeps_per_frame: int = 25
    gravity: tuple[float, float, float] = (0.0, -9.8, 0.0)
    boundary_width: int = 3
    boundary: str = "clamp"
    collision_theta: float | None = None
    accumulation_chunks: int = 8  # accepted for compatibility; GPU order is independent of it
    stress_form: str = "kernel"
    collider_mode: str = "frozen"
    deterministic: bool = False
    rebin_interval: int = 25

    def __post_init__(self):
        if self.dt <= 0.0:
            raise ParameterError("dt must be positive")
        if self.substeps_per_frame < 1:
            raise ParameterError("substeps_per_frame must be >= 1")
        if self.boundary not in ("clamp", "stick"):
            raise ParameterError(f"unknown boundary mode {self.boundary!r}")
        if self.accumulation_chunks < 1:
            raise ParameterError("accumulation_chunks must be >= 1")
        if self.stress_form not in ("kernel", "spec"):
            raise ParameterError(f"unknown stress form {self.stress_form!r}")
        if self.collider_mode not in ("frozen", "live"):
            raise ParameterError(f"unknown collider mode {self.collider_mode!r}")
        if self.rebin_interval < 1:
            raise ParameterError("rebin_interval must be >= 1")


@dataclass
class StepReport:
    step_index: int
    sim_time: float
    timings_ms: dict[str, float]
    inverted_particles: int


def default_device() -> int:
    env = os.environ.get("SOFTMPM_B200_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


class SimState:
    """Particle state + grid of one scene, resident on one B200."""

    def __init__(self, grid: Grid, x, v, F, C, mass, vol0, material_id, time: float = 0.0,
                 step_count: int = 0, device: int | None = None):
        self.grid = grid
        self._h: dict[str, np.ndarray] = {}
        n = len(np.asarray(x))
        shapes = {"x": (n, 3), "v": (n, 3), "F": (n, 3, 3), "C": (n, 3, 3)}
        for name, val in zip(_FIELDS, (x, v, F, C)):
            arr = np.array(val, dtype=np.float64, order="C", copy=True)
            if arr.shape != shapes[name]:
                raise ParameterError(f"SimState.{name} must have shape {shapes[name]}, got {arr.shape}")
            self._h[name] = arr
        self._mass = np.array(mass, dtype=np.float64, copy=True)
        self._vol0 = np.array(vol0, dtype=np.float64, copy=True)
        self._mat = np.array(material_id, dtype=np.int32, copy=True)
        self.time = float(time)
        self.step_count = int(step_count)
        self.device = default_device() if device is None else int(device)
        self._ctx: _lib.Context | None = None
        self._dev_newer: set[str] = set()
        self._host_dirty: set[str] = set(_FIELDS)
        self._static_dirty = True
        nx, ny, nz = grid.resolution
        self._grid_mv = np.zeros((nx, ny, nz, 3))
        self._grid_m = np.zeros((nx, ny, nz))
        self._grid_dev_newer = False
        self._grid_host_dirty = False
        self._cfg_key = None
        self._mat_key = None
        self._packed: PackedColliders | None = None
        self._packed_for: tuple[int, ...] = ()
        self._collision_cache: CollisionField | None = None
        self._collision_src = None
        self._env_tiles = (1, 1, 1)   # set by batch.EnvBatch (BASELINE config 4)
        self._colliders_per_env = 0

    # ---------------------------------------------------------------- fields
    def _get(self, name: str) -> np.ndarray:
        if getattr(self, "_slab_window", False):
            from .errors import SimError
            raise SimError("slab window state: read it through slab.SlabWindow.download()")
        if name in self._dev_newer:
            self._download((name,))
        self._host_dirty.add(name)
        return self._h[name]

    def _set(self, name: str, value) -> None:
        arr = np.array(value, dtype=np.float64, order="C", copy=True)
        if arr.shape != self._h[name].shape:
            self._static_dirty = True  # particle count change -> full re-upload
        self._h[name] = arr
        self._dev_newer.discard(name)
        self._host_dirty.add(name)

    def _adopt(self, name: str, value) -> None:
        """Take the caller's array itself as the host mirror of a field when it
        already has the mirror's layout (C-contiguous, writeable fp64 of the
        same shape): uploads read it and downloads land in it, no copy (the
        drop-in's host-buffer path, install.py); else as _set."""
        if (isinstance(value, np.ndarray) and value.dtype == np.float64 and value.flags.c_contiguous
                and value.flags.writeable and value.shape == self._h[name].shape):
            self._h[name] = value
            self._dev_newer.discard(name)
            self._host_dirty.add(name)
        else:
            self._set(name, value)

    x = property(lambda s: s._get("x"), lambda s, v: s._set("x", v))
    v = property(lambda s: s._get("v"), lambda s, v: s._set("v", v))
    F = property(lambda s: s._get("F"), lambda s, v: s._set("F", v))
    C = property(lambda s: s._get("C"), lambda s, v: s._set("C", v))

    def _static_get(self, attr):
        self._static_dirty = True
        return getattr(self, attr)

    def _static_set(self, attr, value, dtype):
        setattr(self, attr, np.array(value, dtype=dtype, copy=True))
        self._static_dirty = True

    mass = property(lambda s: s._static_get("_mass"),
                    lambda s, v: s._static_set("_mass", v, np.float64))
    vol0 = property(lambda s: s._static_get("_vol0"),
                    lambda s, v: s._static_set("_vol0", v, np.float64))
    material_id = property(lambda s: s._static_get("_mat"),
                           lambda s, v: s._static_set("_mat", v, np.int32))

    @property
    def grid_mv(self) -> np.ndarray:
        self._download_grid()
        self._grid_host_dirty = True
        return self._grid_mv

    @grid_mv.setter
    def grid_mv(self, value):
        self._download_grid()
        self._grid_mv[...] = value
        self._grid_host_dirty = True

    @property
    def grid_m(self) -> np.ndarray:
        self._download_grid()
        self._grid_host_dirty = True
        return self._grid_m

    @grid_m.setter
    def grid_m(self, value):
        self._download_grid()
        self._grid_m[...] = value
        self._grid_host_dirty = True

    @property
    def _collision(self) -> CollisionField | None:
        """Merged field of the last substep's poses (core.py:110; read by demo 02)."""
        if self._collision_cache is None and self._collision_src is not None:
            colliders, theta = self._collision_src
            self._collision_cache = _field_for_state(self, colliders, theta)
        return self._collision_cache

    @_collision.setter
    def _collision(self, value):
        self._collision_cache = value
        self._collision_src = None

    @classmethod
    def from_spawns(cls, grid: Grid, spawns, materials: list[Material]) -> "SimState":
        """core.py:119-143."""
        xs, vols, mats = [], [], []
        lo, hi = grid.margin_bounds()
        for s in spawns:
            pos = np.asarray(s.positions, dtype=np.float64)
            if pos.size == 0:
                raise SpawnError("empty spawn")
            if (pos < lo).any() or (pos > hi).any():
                raise SpawnError("spawned particles violate the 1.5-cell domain margin")
            if not 0 <= s.material_id < len(materials):
                raise SpawnError(f"spawn references material {s.material_id} "
                                 f"but only {len(materials)} are defined")
            xs.append(pos)
            vols.append(np.full(len(pos), s.rest_volume_per_particle))
            mats.append(np.full(len(pos), s.material_id, dtype=np.int32))
        x = np.concatenate(xs)
        vol0 = np.concatenate(vols)
        mat_id = np.concatenate(mats)
        density = np.array([materials[m].density for m in mat_id])
        n = len(x)
        return cls(grid=grid, x=x, v=np.zeros((n, 3)), F=np.tile(np.eye(3), (n, 1, 1)),
                   C=np.zeros((n, 3, 3)), mass=density * vol0, vol0=vol0, material_id=mat_id)

    @property
    def particle_count(self) -> int:
        return len(self._h["x"])

    def has_nan(self) -> bool:
        """core.py:149-151, evaluated on the device when the state lives there."""
        if self._ctx is None or self._host_dirty or self._static_dirty:
            if self._ctx is None:
                return bool(np.isnan(self._h["x"]).any() or np.isnan(self._h["v"]).any()
                            or np.isnan(self._h["F"]).any())
            self._sync_particles()
        flag = ctypes.c_int(0)
        self._ctx.call("mpm_has_nan", ctypes.byref(flag))
        return bool(flag.value)

    # --------------------------------------------------------- device plumbing
    def _config(self, params: SimParams, theta: float | None) -> _lib.MpmConfig:
        g = self.grid
        cfg = _lib.MpmConfig()
        cfg.device = self.device
        cfg.res = (ctypes.c_int * 3)(*g.resolution)
        cfg.dx = g.dx
        cfg.dt = float(params.dt)
        cfg.gravity = (ctypes.c_double * 3)(*[float(a) for a in params.gravity])
        cfg.boundary_width = int(params.boundary_width)
        cfg.stick = int(params.boundary == "stick")
        cfg.theta = -1.0 if theta is None else float(theta)
        cfg.stress_form = 0 if params.stress_form == "kernel" else 1
        cfg.mode_live = int(params.collider_mode == "live")
        cfg.deterministic = int(bool(params.deterministic))
        cfg.rebin_interval = int(params.rebin_interval)
        cfg.env_tiles = (ctypes.c_int * 3)(*self._env_tiles)
        cfg.colliders_per_env = int(self._colliders_per_env)
        return cfg

    def _prepare(self, materials, params: SimParams, theta: float | None = None) -> _lib.Context:
        cfg = self._config(params, theta)
        key = bytes(cfg)
        if self._ctx is None:
            self._ctx = _lib.Context(cfg)
            self._static_dirty = True
        elif key != self._cfg_key:
            self._ctx.call("mpm_set_config", ctypes.byref(cfg))
        self._cfg_key = key
        if materials is not None:
            mu, lam, _ = pack_materials(materials)
            mk = (tuple(mu), tuple(lam))
            if mk != self._mat_key:
                self._ctx.call("mpm_set_materials", _lib.ptr(mu), _lib.ptr(lam), len(mu))
                self._mat_key = mk
            if self._mat.size and (self._mat.min() < 0 or self._mat.max() >= len(mu)):
                raise ParameterError("material_id out of range")
        self._sync_particles()
        return self._ctx

    def _check_margin(self) -> None:
        lo, hi = self.grid.margin_bounds()
        x = self._h["x"]
        if x.size and ((x < lo).any() or (x > hi).any()):
            # mirrors bspline_weights' StencilError; the kernels clamp base cells
            raise StencilError("particle positions leave no room for the 3x3x3 stencil")

    def _sync_particles(self) -> None:
        if getattr(self, "_slab_window", False):
            return  # slab windows own their particle set on the device (migration)
        ctx = self._ctx
        n = len(self._h["x"])
        if self._static_dirty and int(_lib.lib().mpm_particle_count(ctx.h)) == n and self._static_same():
            # a read of mass / vol0 / material_id (the getter cannot know whether
            # the caller wrote into the array) that left them unchanged
            self._static_dirty = False
        if self._static_dirty or int(_lib.lib().mpm_particle_count(ctx.h)) != n:
            for name in list(self._dev_newer):
                self._download((name,))
            if "x" in self._host_dirty:
                self._check_margin()
            ctx.call("mpm_upload_particles", ctypes.c_int64(n), _lib.ptr(self._h["x"]),
                     _lib.ptr(self._h["v"]), _lib.ptr(self._h["F"]), _lib.ptr(self._h["C"]),
                     _lib.ptr(np.ascontiguousarray(self._mass)),
                     _lib.ptr(np.ascontiguousarray(self._vol0)),
                     _lib.ptr(np.ascontiguousarray(self._mat), _lib._I32))
            self._static_dirty = False
            self._static_snap = (self._mass.copy(), self._vol0.copy(), self._mat.copy())
            self._host_dirty.clear()
            return
        if self._host_dirty:
            if "x" in self._host_dirty:
                self._check_margin()
            mask = 0
            arrs = {}
            for name in _FIELDS:
                if name in self._host_dirty:
                    mask |= _FIELD_BIT[name]
                    arrs[name] = self._h[name]
            ctx.call("mpm_upload_fields", ctypes.c_uint32(mask),
                     *[_lib.ptr(arrs.get(nm)) for nm in _FIELDS])
            self._host_dirty.clear()

    def _static_same(self) -> bool:
        snap = getattr(self, "_static_snap", None)
        return snap is not None and all(
            a.shape == b.shape and np.array_equal(a, b)
            for a, b in zip(snap, (self._mass, self._vol0, self._mat)))

    def _download(self, names) -> None:
        mask = _KEEP_EQUAL
        for nm in names:
            mask |= _FIELD_BIT[nm]
        # in place (callers may hold the arrays); the device holds fp32: where
        # its value is the fp32 rounding of the host's last value (the kernels
        # left it unchanged), the host's fp64 value is kept instead of the
        # rounded one (e.g. G2P with a zero velocity field leaves x
        # bit-identical, test_transfers.py:121) -- merged on the library's
        # host threads (MPM_DOWNLOAD_KEEP_EQUAL)
        self._ctx.call("mpm_download_particles", ctypes.c_uint32(mask),
                       *[_lib.ptr(self._h[nm] if nm in names else None) for nm in _FIELDS])
        for nm in names:
            self._dev_newer.discard(nm)

    def _download_grid(self) -> None:
        if self._grid_dev_newer:
            self._ctx.call("mpm_download_grid", _lib.ptr(self._grid_mv), _lib.ptr(self._grid_m))
            self._grid_dev_newer = False

    def _upload_grid(self, target: int) -> None:
        if self._grid_host_dirty:
            self._ctx.call("mpm_upload_grid", target, _lib.ptr(self._grid_mv),
                           _lib.ptr(self._grid_m if target == 0 else None))
            self._grid_host_dirty = False

    def _device_wrote(self, names, grid: bool = True) -> None:
        for nm in names:
            self._dev_newer.add(nm)
            self._host_dirty.discard(nm)
        if grid:
            self._grid_dev_newer = True
            self._grid_host_dirty = False

    def _packed_colliders(self, colliders: list[RigidCollider],
                          params: SimParams | None = None) -> PackedColliders | None:
        """Pack on first use / identity change, else refresh poses only (core.py:160-169)."""
        if not colliders:
            return None
        key = tuple(id(c) for c in colliders)
        if self._packed is None or self._packed_for != key:
            self._packed = pack_colliders(colliders)
            self._packed_for = key
            self._packed_uploaded = False
        else:
            self._packed.refresh_poses(colliders)
            if params is not None and params.collider_mode == "live":
                self._packed.mode[:] = [MODE_NAMES[c.mode] for c in colliders]
        return self._packed

    def _upload_colliders(self) -> None:
        p = self._packed
        if not getattr(self, "_packed_uploaded", False):
            sdf = np.ascontiguousarray(p.sdf_values, np.float64)
            self._ctx.call("mpm_set_colliders", len(p.kind), _lib.ptr(p.kind, _lib._I32),
                           _lib.ptr(p.half), _lib.ptr(p.rotation), _lib.ptr(p.translation),
                           _lib.ptr(p.linear_velocity), _lib.ptr(p.angular_velocity),
                           _lib.ptr(p.friction), _lib.ptr(p.mode, _lib._I32), _lib.ptr(sdf),
                           ctypes.c_int64(sdf.size), _lib.ptr(p.sdf_offset, _lib._I64),
                           _lib.ptr(p.sdf_resolution, _lib._I32), _lib.ptr(p.sdf_bounds_min),
                           _lib.ptr(p.sdf_extent))
            self._packed_uploaded = True

    def _upload_pose_rows(self, R, T, lv, av, mode) -> None:
        self._ctx.call("mpm_set_pose_table", len(R), _lib.ptr(R), _lib.ptr(T), _lib.ptr(lv),
                       _lib.ptr(av), _lib.ptr(mode, _lib._I32))

    @property
    def launches(self) -> int:
        return 0 if self._ctx is None else self._ctx.launches


# ---------------------------------------------------------------------------
# stencil weights (host utility, core.py:176-194)
# ---------------------------------------------------------------------------

def bspline_weights(xp: np.ndarray, grid: Grid) -> tuple[np.ndarray, np.ndarray]:
    xp = np.asarray(xp, dtype=np.float64)
    xg = xp / grid.dx
    base = np.floor(xg - 0.5).astype(np.int64)
    if (base < 0).any() or (base + 2 >= np.array(grid.resolution)).any():
        raise StencilError(f"position {xp} leaves no room for its 3x3x3 stencil")
    f = xg - base
    w = np.empty((3, 3))
    w[:, 0] = 0.5 * (1.5 - f) ** 2
    w[:, 1] = 0.75 - (f - 1.0) ** 2
    w[:, 2] = 0.5 * (f - 0.5) ** 2
    return base, w


# ---------------------------------------------------------------------------
# pipeline stages (core.py:211-258)
# ---------------------------------------------------------------------------

def _theta(state: SimState, params: SimParams) -> float:
    return params.collision_theta if params.collision_theta is not None else 0.5 * state.grid.dx


def _pose_arrays(packed: PackedColliders):
    return (np.ascontiguousarray(packed.rotation[None]), np.ascontiguousarray(packed.translation[None]),
            np.ascontiguousarray(packed.linear_velocity[None]),
            np.ascontiguousarray(packed.angular_velocity[None]),
            np.ascontiguousarray(packed.mode[None], np.int32))


def p2g(state: SimState, materials: list[Material], params: SimParams) -> int:
    """Scatter momentum/mass to the grid; F advanced in place; returns the det<=0 count."""
    ctx = state._prepare(materials, params)
    inv = ctypes.c_int64(0)
    state._grid_host_dirty = False  # p2g overwrites every node (kernels.py:317-340)
    ctx.call("mpm_p2g", ctypes.byref(inv))
    state._device_wrote(("F",))
    return int(inv.value)


def grid_update(state: SimState, params: SimParams, collision: CollisionField | None = None,
                colliders: list[RigidCollider] | None = None) -> None:
    """Momentum -> velocity, gravity, collision, domain boundary (core.py:228-251)."""
    colliders = colliders or []
    use = collision is not None and bool(colliders)
    ctx = state._prepare(None, params, collision.theta if use else None)
    if use:
        packed = state._packed_colliders(colliders, params)
        state._upload_colliders()
        state._upload_pose_rows(*_pose_arrays(packed))
    state._upload_grid(0)
    ctx.call("mpm_grid_update", int(use))
    state._grid_dev_newer = True


def g2p_advect(state: SimState, params: SimParams) -> None:
    """Gather velocities, rebuild C, advect, clamp (core.py:254-258)."""
    ctx = state._prepare(None, params)
    state._upload_grid(1)
    ctx.call("mpm_g2p")
    state._device_wrote(("x", "v", "C"), grid=False)


def _run_substeps(state: SimState, materials, params: SimParams, colliders, nsub: int,
                  pose_rows) -> tuple[int, float]:
    theta = _theta(state, params) if colliders else None
    ctx = state._prepare(materials, params, theta)
    if colliders:
        state._upload_colliders()
        state._upload_pose_rows(*pose_rows)
    state._grid_host_dirty = False
    inv = ctypes.c_int64(0)
    dev_ms = ctypes.c_double(0.0)
    ctx.call("mpm_substeps", nsub, int(bool(colliders)), ctypes.byref(inv), ctypes.byref(dev_ms))
    state._device_wrote(_FIELDS)
    state._collision_cache = None
    state._collision_src = (list(colliders), theta) if colliders else None
    return int(inv.value), float(dev_ms.value)


class _Upload:
    """SimState._prepare (context config, materials, host-dirty field upload)
    on a worker thread; join() re-raises its error on the caller's thread."""

    def __init__(self, state, materials, params, theta):
        import threading
        self.err = None

        def run():
            try:
                state._prepare(materials, params, theta)
            except BaseException as e:  # noqa: BLE001 -- handed to the caller
                self.err = e

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()

    def join(self):
        self.t.join()
        if self.err is not None:
            raise self.err


def substep(state: SimState, materials: list[Material], params: SimParams,
            colliders: list[RigidCollider] | None = None) -> int:
    """One substep (core.py:261-277); returns the inverted-element count."""
    colliders = colliders or []
    rows = None
    if colliders:
        rows = _pose_arrays(state._packed_colliders(colliders, params))
    inv, _ = _run_substeps(state, materials, params, colliders, 1, rows)
    state.time += params.dt
    return inv


def pose_table(state: SimState, colliders: list[RigidCollider], params: SimParams, pose_fn, t0: float):
    """Per-substep collider pose table of one frame: ``pose_fn(colliders, t)``
    at t0, t0 + dt, ... (core.py:296-303; times accumulated like the
    reference's loop), packed as core.step uploads it.  A ``make_pose_fn``
    feed evaluates the whole frame at once (scene.PoseFn.table); any other
    callable is called once per substep."""
    nsub = params.substeps_per_frame
    times, t = [], t0
    for _ in range(nsub):
        times.append(t)
        t += params.dt
    table = getattr(pose_fn, "table", None)
    if table is None:
        R, T, lv, av, md = [], [], [], [], []
        for t in times:
            pose_fn(colliders, t)
            pk = state._packed_colliders(colliders, params)
            R.append(pk.rotation.copy())
            T.append(pk.translation.copy())
            lv.append(pk.linear_velocity.copy())
            av.append(pk.angular_velocity.copy())
            md.append(pk.mode.copy())
        return (np.ascontiguousarray(R), np.ascontiguousarray(T), np.ascontiguousarray(lv),
                np.ascontiguousarray(av), np.ascontiguousarray(md, np.int32))
    if state._packed is None or state._packed_for != tuple(id(c) for c in colliders):
        pose_fn(colliders, times[0])  # first pack sees the first substep's modes (F7)
        state._packed_colliders(colliders, params)
    R, T, lv, av, modes = table(colliders, times)
    pk = state._packed_colliders(colliders, params)  # colliders now at the last substep's pose
    if params.collider_mode == "live":
        md = np.array([[MODE_NAMES[m] for m in row] for row in modes], dtype=np.int32)
    else:
        md = np.repeat(pk.mode[None].astype(np.int32), nsub, axis=0)
    return (np.ascontiguousarray(R), np.ascontiguousarray(T), np.ascontiguousarray(lv),
            np.ascontiguousarray(av), np.ascontiguousarray(md, np.int32))


def step(state: SimState, materials: list[Material], params: SimParams,
         colliders: list[RigidCollider] | None = None, pose_fn=None) -> StepReport:
    """One frame of ``substeps_per_frame`` substeps (core.py:280-320)."""
    colliders = colliders or []
    nsub = params.substeps_per_frame
    t_collision = 0.0
    rows = None
    upload = None
    if colliders and state._ctx is not None and state._host_dirty and not state._static_dirty:
        # host-modified fields go up on a worker thread (the copy releases the
        # GIL) while this thread builds the frame's pose table; pose_fn itself
        # stays on the caller's thread
        upload = _Upload(state, materials, params, _theta(state, params))
    if colliders:
        t0 = _time.perf_counter()
        if pose_fn is not None:
            rows = pose_table(state, colliders, params, pose_fn, state.time)
        else:
            rows = _pose_arrays(state._packed_colliders(colliders, params))
        t_collision += _time.perf_counter() - t0
    t0 = _time.perf_counter()
    if upload is not None:
        upload.join()
    inv, _ = _run_substeps(state, materials, params, colliders, nsub, rows)
    t_soft = _time.perf_counter() - t0
    for _ in range(nsub):
        state.time += params.dt
    state.step_count += 1
    return StepReport(step_index=state.step_count, sim_time=state.time,
                      timings_ms={"collision_detection": 1000.0 * t_collision,
                                  "soft_simulation": 1000.0 * t_soft},
                      inverted_particles=inv)


# ---------------------------------------------------------------------------
# collision-field evaluation on the device
# ---------------------------------------------------------------------------

_FIELD_CTX: dict = {}


def _field_ctx(grid: Grid) -> _lib.Context:
    key = (grid.resolution, grid.dx, default_device())
    ctx = _FIELD_CTX.get(key)
    if ctx is None:
        st = SimState(grid, np.zeros((1, 3)), np.zeros((1, 3)), np.zeros((1, 3, 3)),
                      np.zeros((1, 3, 3)), np.ones(1), np.ones(1), np.zeros(1, np.int32))
        cfg = st._config(SimParams(), None)
        ctx = _lib.Context(cfg)
        _FIELD_CTX[key] = ctx
    return ctx


def _set_colliders_on(ctx: _lib.Context, packed: PackedColliders) -> None:
    sdf = np.ascontiguousarray(packed.sdf_values, np.float64)
    ctx.call("mpm_set_colliders", len(packed.kind), _lib.ptr(packed.kind, _lib._I32),
             _lib.ptr(np.ascontiguousarray(packed.half)), _lib.ptr(np.ascontiguousarray(packed.rotation)),
             _lib.ptr(np.ascontiguousarray(packed.translation)),
             _lib.ptr(np.ascontiguousarray(packed.linear_velocity)),
             _lib.ptr(np.ascontiguousarray(packed.angular_velocity)),
             _lib.ptr(np.ascontiguousarray(packed.friction)), _lib.ptr(packed.mode, _lib._I32),
             _lib.ptr(sdf), ctypes.c_int64(sdf.size), _lib.ptr(packed.sdf_offset, _lib._I64),
             _lib.ptr(packed.sdf_resolution, _lib._I32),
             _lib.ptr(np.ascontiguousarray(packed.sdf_bounds_min)),
             _lib.ptr(np.ascontiguousarray(packed.sdf_extent)))


def _field_on_device(grid: Grid, packed: PackedColliders, theta: float):
    ctx = _field_ctx(grid)
    _set_colliders_on(ctx, packed)
    dist = np.empty(grid.resolution)
    obj = np.empty(grid.resolution, dtype=np.int32)
    ctx.call("mpm_collision_field", ctypes.c_double(theta), _lib.ptr(dist), _lib.ptr(obj, _lib._I32))
    return dist, obj


def _field_for_state(state: SimState, colliders, theta: float) -> CollisionField:
    dist, obj = _field_on_device(state.grid, pack_colliders(colliders), theta)
    return CollisionField(distance=dist, object_id=obj, theta=theta)
