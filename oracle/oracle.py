"""ctypes front end of the CPU oracle (``liboracle.so``, built from mpm_oracle.c).

TEST INFRASTRUCTURE ONLY.  Importable from ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``; the
product package never imports this module.

O1 = fp64 restatement of the reference numba kernels
     (/root/reference/pkg/src/softmpm/kernels.py:161-534, core.py:211-320);
O2 = fp64 loop-nest spec oracle (reference.py:14-200);
O3 = fp32 deterministic-order P2G (the order the GPU deterministic mode uses).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "mpm_oracle.c")):
        subprocess.run(["make", "-C", _HERE, "-B" if force else "liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_substep.restype = ctypes.c_int64
        _lib.orc_max_threads.restype = ctypes.c_int
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(ctypes.c_int(int(n)))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _p(a, kind=_D):
    return a.ctypes.data_as(kind)


def _c64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


@dataclass
class OracleParams:
    res: tuple[int, int, int]
    dx: float
    dt: float = 5.0e-4
    gravity: tuple[float, float, float] = (0.0, -9.8, 0.0)
    boundary_width: int = 3
    stick: bool = False
    theta: float = -1.0
    chunks: int = 8
    stress_form: int = 0  # 0 = kernel (F^-1, drop-in parity), 1 = spec (F^-T)

    @property
    def hi(self):
        return tuple((r - 1.5 - 1.0e-7) * self.dx for r in self.res)


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("dx", ctypes.c_double), ("dt", ctypes.c_double),
                ("gx", ctypes.c_double), ("gy", ctypes.c_double), ("gz", ctypes.c_double),
                ("bwidth", ctypes.c_int), ("stick", ctypes.c_int),
                ("theta", ctypes.c_double), ("hi", ctypes.c_double * 3),
                ("nchunks", ctypes.c_int), ("stress_form", ctypes.c_int)]


def empty_packed():
    """Collider tables with zero colliders, shaped like collision.PackedColliders."""
    return dict(kind=np.zeros(0, np.int32), half=np.zeros((0, 3)), rotation=np.zeros((0, 3, 3)),
                translation=np.zeros((0, 3)), linear_velocity=np.zeros((0, 3)),
                angular_velocity=np.zeros((0, 3)), friction=np.zeros(0),
                mode=np.zeros(0, np.int32), sdf_values=np.zeros(1), sdf_offset=np.zeros(0, np.int64),
                sdf_resolution=np.zeros((0, 3), np.int32), sdf_bounds_min=np.zeros((0, 3)),
                sdf_extent=np.ones(0))


def _packed_args(packed):
    """Flatten a PackedColliders-like object (reference or ours) to C arrays."""
    if packed is None:
        packed = empty_packed()
    get = (lambda k: packed[k]) if isinstance(packed, dict) else (lambda k: getattr(packed, k))
    arrs = dict(
        kind=np.ascontiguousarray(get("kind"), np.int32),
        half=_c64(get("half")), rotation=_c64(get("rotation")),
        translation=_c64(get("translation")), linear_velocity=_c64(get("linear_velocity")),
        angular_velocity=_c64(get("angular_velocity")), friction=_c64(get("friction")),
        mode=np.ascontiguousarray(get("mode"), np.int32), sdf_values=_c64(get("sdf_values")),
        sdf_offset=np.ascontiguousarray(get("sdf_offset"), np.int64),
        sdf_resolution=np.ascontiguousarray(get("sdf_resolution"), np.int32),
        sdf_bounds_min=_c64(get("sdf_bounds_min")), sdf_extent=_c64(get("sdf_extent")))
    if arrs["sdf_values"].size == 0:
        arrs["sdf_values"] = np.zeros(1)
    return arrs


class OracleSim:
    """fp64 CPU substep over caller-owned numpy state (the O1 oracle).

    Mirrors softmpm.core.substep/step (core.py:261-320): p2g_scatter +
    p2g_reduce, collision field over all nodes, grid_update, g2p_advect, with
    the reference's fixed-chunk accumulation.  State arrays are updated in
    place; grid_mv/grid_m hold the last substep's grid like SimState does.
    """

    def __init__(self, params: OracleParams, x, v, F, C, mass, vol0, material_id, mu, lam):
        self.p = params
        self.x = _c64(x).copy()
        self.v = _c64(v).copy()
        self.F = _c64(F).copy()
        self.C = _c64(C).copy()
        self.mass = _c64(mass)
        self.vol0 = _c64(vol0)
        self.material_id = np.ascontiguousarray(material_id, np.int32)
        self.mu = _c64(np.atleast_1d(mu))
        self.lam = _c64(np.atleast_1d(lam))
        nx, ny, nz = params.res
        nn = nx * ny * nz
        self.grid_mv = np.zeros((nx, ny, nz, 3))
        self.grid_m = np.zeros((nx, ny, nz))
        self._buf = np.zeros((max(1, params.chunks), nn, 4))
        self._dist = np.zeros(nn)
        self._obj = np.zeros(nn, np.int32)
        self.time = 0.0

    def substep(self, packed=None) -> int:
        p = self.p
        cp = _packed_args(packed)
        ncol = len(cp["kind"])
        prm = _Params(p.res[0], p.res[1], p.res[2], p.dx, p.dt, *p.gravity, p.boundary_width,
                      int(p.stick), p.theta if ncol else -1.0, (ctypes.c_double * 3)(*p.hi),
                      p.chunks, p.stress_form)
        n = len(self.x)
        inv = lib().orc_substep(
            ctypes.byref(prm), ctypes.c_long(n), _p(self.x), _p(self.v), _p(self.F), _p(self.C),
            _p(self.mass), _p(self.vol0), _p(self.material_id, _I32), _p(self.mu), _p(self.lam),
            _p(self.grid_mv), _p(self.grid_m), _p(self._buf), _p(self._dist),
            _p(self._obj, _I32), ctypes.c_int(ncol), _p(cp["kind"], _I32), _p(cp["half"]),
            _p(cp["rotation"]), _p(cp["translation"]), _p(cp["linear_velocity"]),
            _p(cp["angular_velocity"]), _p(cp["friction"]), _p(cp["mode"], _I32),
            _p(cp["sdf_values"]), _p(cp["sdf_offset"], _I64), _p(cp["sdf_resolution"], _I32),
            _p(cp["sdf_bounds_min"]), _p(cp["sdf_extent"]))
        self.time += p.dt
        return int(inv)

    def collision_field(self, packed, theta):
        cp = _packed_args(packed)
        nx, ny, nz = self.p.res
        dist = np.zeros((nx, ny, nz))
        obj = np.zeros((nx, ny, nz), np.int32)
        lib().orc_build_collision_field(
            ctypes.c_double(self.p.dx), nx, ny, nz, _p(dist), _p(obj, _I32),
            ctypes.c_double(2.0 * theta), ctypes.c_int(len(cp["kind"])), _p(cp["kind"], _I32),
            _p(cp["half"]), _p(cp["rotation"]), _p(cp["translation"]), _p(cp["sdf_values"]),
            _p(cp["sdf_offset"], _I64), _p(cp["sdf_resolution"], _I32),
            _p(cp["sdf_bounds_min"]), _p(cp["sdf_extent"]))
        return dist, obj


def reference_substep(x, v, F, C, mass, vol0, material_id, mu, lam, grid_mv, grid_m, dt, dx,
                      gravity, bwidth, stick, hi):
    """O2: loop-nest spec-form substep (reference.py:14-200), arrays in place."""
    nx, ny, nz = grid_m.shape
    for a in (x, v, F, C, grid_mv, grid_m):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    lib().orc_reference_substep(
        ctypes.c_long(len(x)), _p(x), _p(v), _p(F), _p(C), _p(_c64(mass)), _p(_c64(vol0)),
        _p(np.ascontiguousarray(material_id, np.int32), _I32), _p(_c64(np.atleast_1d(mu))),
        _p(_c64(np.atleast_1d(lam))), _p(grid_mv), _p(grid_m), nx, ny, nz,
        ctypes.c_double(dt), ctypes.c_double(dx), ctypes.c_double(gravity[0]),
        ctypes.c_double(gravity[1]), ctypes.c_double(gravity[2]), ctypes.c_int(bwidth),
        ctypes.c_int(int(stick)), ctypes.c_double(hi[0]), ctypes.c_double(hi[1]),
        ctypes.c_double(hi[2]))


def p2g_sorted_fp32(x, v, F, C, mass, vol0, material_id, mu, lam, dt, dx, res, order,
                    stress_form=0):
    """O3: fp32 P2G scattered in ``order`` (ascending base-cell key, then index).

    Returns (grid_mv (nx,ny,nz,3) f32, grid_m (nx,ny,nz) f32, F' (n,3,3) f32, inverted).
    """
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    x, v, C, mass, vol0 = map(f32, (x, v, C, mass, vol0))
    F = f32(F).copy()
    nx, ny, nz = res
    gmv = np.zeros((nx, ny, nz, 3), np.float32)
    gm = np.zeros((nx, ny, nz), np.float32)
    inv = ctypes.c_int64(0)
    order = np.ascontiguousarray(order, np.int64)
    lib().orc32_p2g_sorted(
        ctypes.c_long(len(x)), _p(order, _I64), _p(x, _F), _p(v, _F), _p(F, _F), _p(C, _F),
        _p(mass, _F), _p(vol0, _F), _p(np.ascontiguousarray(material_id, np.int32), _I32),
        _p(f32(np.atleast_1d(mu)), _F), _p(f32(np.atleast_1d(lam)), _F), ctypes.c_float(dt),
        ctypes.c_float(dx), ctypes.c_int(nx), ctypes.c_int(ny), ctypes.c_int(nz), _p(gmv, _F),
        _p(gm, _F),
        ctypes.c_int(stress_form), ctypes.byref(inv))
    return gmv, gm, F, int(inv.value)


def sorted_order(x32, dx, res):
    """Ascending (base-cell key, original index) permutation of fp32 positions."""
    x32 = np.ascontiguousarray(x32, np.float32)
    inv_dx = np.float32(1.0) / np.float32(dx)
    b = np.floor(x32 * inv_dx - np.float32(0.5)).astype(np.int64)
    b = np.clip(b, 0, np.asarray(res) - 3)
    key = (b[:, 0] * res[1] + b[:, 1]) * res[2] + b[:, 2]
    return np.lexsort((np.arange(len(x32)), key))


def splat_density(positions, masses, res, dx, chunks: int = 8):
    """surfacing.splat_density (surfacing.py:45-67 -> kernels.py:541-588):
    dense (res0, res1, res2) fp64 mass density, chunked like the reference."""
    res = tuple(int(r) for r in res)
    nn = res[0] * res[1] * res[2]
    pos = _c64(positions).reshape(-1, 3)
    m = _c64(masses).reshape(-1)
    buf = np.zeros((chunks, nn))
    out = np.zeros(res)
    L = lib()
    if len(pos):
        L.orc_splat_mass(ctypes.c_long(len(pos)), _p(pos), _p(m), ctypes.c_double(dx), res[0], res[1], res[2],
                         _p(buf), ctypes.c_int(chunks))
    L.orc_splat_reduce(_p(buf), _p(out), ctypes.c_long(nn), ctypes.c_int(chunks), ctypes.c_double(1.0 / dx ** 3))
    return out


def compute_metrics(x, F, x0, dx):
    """scene.compute_metrics (scene.py:204-220), the same numpy expressions:
    (lifted_fraction, detached_fraction, mean |det F - 1|, max displacement)."""
    x = np.asarray(x, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    dy = x[:, 1] - x0[:, 1]
    j = np.linalg.det(np.asarray(F, dtype=np.float64))
    disp = np.linalg.norm(x - x0, axis=1)
    return (float((dy > 2.0 * dx).mean()), float((dy > dx).mean()), float(np.abs(j - 1.0).mean()),
            float(disp.max() if len(disp) else 0.0))
