"""Per-frame consumers of the particle state, on the device.

* ``compute_metrics(state, initial_positions)`` -- scene.py:190-220
  (``MetricSample`` / ``compute_metrics``): lifted / detached fractions,
  mean |det F - 1| and max displacement as one device reduction instead of a
  download of x and F (cli.py:86 calls it every frame).
* ``splat_density(positions, masses, grid, resolution)`` -- surfacing.py:45-67
  (-> kernels.splat_mass / splat_reduce, kernels.py:541-588): the
  quadratic B-spline mass deposit that feeds marching cubes, on the GPU;
  ``density_field(state, resolution)`` splats a SimState's own particles
  without downloading them.
* ``marching_cubes(field, iso)`` / ``compute_uvs`` / ``extract_surface`` --
  surfacing.py:70-112: the isosurface on the GPU (case table derived in
  tools/gen_mc_table.py; the reference calls scikit-image's Lorensen tables,
  absent here, so triangle-level parity is not pinned -- the tests check the
  reference's own geometric cases and watertightness); ``extract_surface``
  splats and triangulates on the device and reads back only the mesh.

All of it runs through the C ABI (``mpm_metrics``, ``mpm_splat_density[_host]``,
``mpm_marching_cubes``, ``mpm_mesh_fetch``); there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import Grid, SimParams, SimState, default_device
from .errors import ParameterError


@dataclass
class MetricSample:
    """scene.py:190-201."""

    time: float
    lifted_fraction: float
    detached_fraction: float
    mean_abs_j_minus_1: float
    max_displacement: float

    def csv_row(self) -> str:
        return (f"{self.time:.6f},{self.lifted_fraction:.6f},"
                f"{self.detached_fraction:.6f},{self.mean_abs_j_minus_1:.8f},"
                f"{self.max_displacement:.6f}")


@dataclass
class ScalarField:
    """surfacing.py:21-26: dense nodal samples (mass density, kg/m^3)."""

    values: np.ndarray
    dx: float


def _device_state(state: SimState) -> _lib.Context:
    """The state's context with the host mirrors pushed (creates one if the
    state has never been stepped)."""
    if state._ctx is None:
        return state._prepare(None, SimParams())
    if state._host_dirty or state._static_dirty:
        state._sync_particles()
    return state._ctx


def _fingerprint(a: np.ndarray) -> tuple:
    step = max(1, len(a) // 97)
    return (a.ctypes.data, a.shape, float(a[::step].sum()), float(a[-1].sum()) if len(a) else 0.0)


def compute_metrics(state: SimState, initial_positions: np.ndarray) -> MetricSample:
    """Deformation/displacement summary relative to the spawn configuration
    (scene.py:204-220): lifted/detached count particles that rose more than
    2 dx / 1 dx above their own spawn height; mean |J - 1| averages volume
    change over particles."""
    x0 = np.ascontiguousarray(initial_positions, dtype=np.float64)
    n = state.particle_count
    if x0.shape != (n, 3):
        raise ParameterError(f"initial_positions must have shape ({n}, 3)")
    out = (ctypes.c_double * 5)()
    if n == 0:
        return MetricSample(state.time, float("nan"), float("nan"), float("nan"), 0.0)
    ctx = _device_state(state)
    key = _fingerprint(x0)
    upload = getattr(state, "_metrics_x0_key", None) != key
    ctx.call("mpm_metrics", _lib.ptr(x0) if upload else _lib.ptr(None), ctypes.c_double(state.grid.dx), out)
    state._metrics_x0_key = key
    return MetricSample(time=state.time, lifted_fraction=out[0], detached_fraction=out[1],
                        mean_abs_j_minus_1=out[2], max_displacement=out[3])


def _field_geometry(grid: Grid, resolution):
    res = tuple(int(r) for r in resolution) if resolution is not None else tuple(grid.resolution)
    dxs = [e / r for e, r in zip(grid.extent, res)]
    if max(dxs) - min(dxs) > 1.0e-12 * max(dxs):
        raise ParameterError("field cell size must be uniform across axes")
    return res, dxs[0]


def splat_density(positions: np.ndarray, masses: np.ndarray, grid: Grid,
                  resolution: tuple[int, int, int] | None = None, chunks: int = 8,
                  device: int | None = None) -> ScalarField:
    """Deposit particle mass on a lattice via the quadratic B-spline stencil
    (surfacing.py:45-67); ``chunks`` is accepted for signature compatibility
    (the reference's CPU determinism scheme)."""
    del chunks
    res, dx = _field_geometry(grid, resolution)
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    m = np.ascontiguousarray(masses, dtype=np.float64).reshape(-1)
    if len(pos) != len(m):
        raise ParameterError("positions and masses differ in length")
    out = np.zeros(res)
    r = (ctypes.c_int32 * 3)(*res)
    L = _lib.lib()
    dev = default_device() if device is None else int(device)
    _lib.check(L.mpm_splat_density_host(dev, _lib.ptr(pos), _lib.ptr(m), ctypes.c_int64(len(pos)), r,
                                        ctypes.c_double(dx), _lib.ptr(out)), None, "mpm_splat_density_host")
    return ScalarField(values=out, dx=dx)


def density_field(state: SimState, resolution: tuple[int, int, int] | None = None) -> ScalarField:
    """``splat_density(state.x, state.mass, state.grid, resolution)`` straight
    from the device-resident particles (no download of x)."""
    res, dx = _field_geometry(state.grid, resolution)
    out = np.zeros(res)
    if state.particle_count == 0:
        return ScalarField(values=out, dx=dx)
    ctx = _device_state(state)
    r = (ctypes.c_int32 * 3)(*res)
    ctx.call("mpm_splat_density", _lib.ptr(None), _lib.ptr(None), ctypes.c_int64(0), r, ctypes.c_double(dx),
             _lib.ptr(out))
    return ScalarField(values=out, dx=dx)


@dataclass
class SurfaceMesh:
    """surfacing.py:29-40."""

    vertices: np.ndarray
    indices: np.ndarray
    uvs: np.ndarray | None = None
    normals: np.ndarray | None = None

    @classmethod
    def empty(cls) -> "SurfaceMesh":
        return cls(vertices=np.zeros((0, 3)), indices=np.zeros((0, 3), dtype=np.int32),
                   uvs=np.zeros((0, 2)), normals=np.zeros((0, 3)))


def _fetch_mesh(ctx: _lib.Context, nv: int, nt: int) -> SurfaceMesh:
    verts = np.zeros((nv, 3))
    normals = np.zeros((nv, 3))
    tris = np.zeros((nt, 3), dtype=np.int32)
    ctx.call("mpm_mesh_fetch", _lib.ptr(verts), _lib.ptr(tris, _lib._I32), _lib.ptr(normals))
    return SurfaceMesh(vertices=verts, indices=tris, normals=normals)


def marching_cubes(fld: ScalarField, iso: float) -> SurfaceMesh:
    """Isosurface of a density field (surfacing.py:70-95): ParameterError for
    iso <= 0, an empty mesh when the field never reaches the iso level."""
    if iso <= 0.0:
        raise ParameterError("iso level must be positive")
    values = np.ascontiguousarray(fld.values, dtype=np.float64)
    vmax = float(values.max()) if values.size else 0.0
    if vmax < iso or float(values.min()) >= iso:
        return SurfaceMesh.empty()
    from .core import _field_ctx
    ctx = _field_ctx(Grid((8, 8, 8)))
    r = (ctypes.c_int32 * 3)(*values.shape)
    nv, nt = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("mpm_marching_cubes", _lib.ptr(values), r, ctypes.c_double(fld.dx), ctypes.c_double(iso),
             ctypes.byref(nv), ctypes.byref(nt))
    return _fetch_mesh(ctx, nv.value, nt.value)


def compute_uvs(mesh: SurfaceMesh, domain_extent) -> SurfaceMesh:
    """Planar top-down projection (surfacing.py:98-106)."""
    ext = np.asarray(domain_extent, dtype=np.float64)
    if len(mesh.vertices):
        u = np.clip(mesh.vertices[:, 0] / ext[0], 0.0, 1.0)
        w = np.clip(mesh.vertices[:, 2] / ext[2], 0.0, 1.0)
        mesh.uvs = np.stack([u, w], axis=1)
    else:
        mesh.uvs = np.zeros((0, 2))
    return mesh


def extract_surface(state: SimState, iso: float, resolution=None) -> SurfaceMesh:
    """splat -> marching cubes -> UVs (surfacing.py:109-112), with the splat
    and the triangulation on the device: only the mesh is read back."""
    if iso <= 0.0:
        raise ParameterError("iso level must be positive")
    res, dx = _field_geometry(state.grid, resolution)
    if state.particle_count == 0:
        return compute_uvs(SurfaceMesh.empty(), state.grid.extent)
    ctx = _device_state(state)
    r = (ctypes.c_int32 * 3)(*res)
    ctx.call("mpm_splat_density", _lib.ptr(None), _lib.ptr(None), ctypes.c_int64(0), r, ctypes.c_double(dx),
             _lib.ptr(None))
    nv, nt = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("mpm_marching_cubes", _lib.ptr(None), _lib.ptr(None, _lib._I32), ctypes.c_double(dx),
             ctypes.c_double(iso), ctypes.byref(nv), ctypes.byref(nt))
    return compute_uvs(_fetch_mesh(ctx, nv.value, nt.value), state.grid.extent)


def export_obj(mesh: SurfaceMesh, path) -> None:
    """Wavefront OBJ of a surface mesh (surfacing.py:115-116): `v` lines, then
    `vt` / `vn` when present (parallel to the vertices), 1-based faces with
    the matching v/vt/vn references."""
    from pathlib import Path
    v = np.asarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(mesh.indices, dtype=np.int64).reshape(-1, 3) + 1
    parts = ["\n".join(f"v {a:.9g} {b:.9g} {c:.9g}" for a, b, c in v)]
    has_t = mesh.uvs is not None and len(mesh.uvs) == len(v)
    has_n = mesh.normals is not None and len(mesh.normals) == len(v)
    if has_t:
        parts.append("\n".join(f"vt {a:.9g} {b:.9g}" for a, b in np.asarray(mesh.uvs).reshape(-1, 2)))
    if has_n:
        parts.append("\n".join(f"vn {a:.9g} {b:.9g} {c:.9g}" for a, b, c in np.asarray(mesh.normals).reshape(-1, 3)))
    tag = "{0}/{0}/{0}" if has_t and has_n else "{0}/{0}" if has_t else "{0}//{0}" if has_n else "{0}"
    parts.append("\n".join("f " + " ".join(tag.format(i) for i in tri) for tri in f))
    Path(path).write_text("\n".join(p for p in parts if p) + "\n", encoding="utf-8")
