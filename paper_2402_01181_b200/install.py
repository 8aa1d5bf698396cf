"""Route the reference package's hot path through the B200 kernels.

``install(softmpm)`` rebinds ``softmpm.core.p2g / grid_update / g2p_advect /
substep / step``, the surfacing consumers ``softmpm.surfacing.splat_density /
marching_cubes / extract_surface`` and ``softmpm.scene.compute_metrics`` --
every binding of them in the loaded package, including the copies that
``from .core import step`` made in ``softmpm.cli`` and ``softmpm.server`` --
so unmodified callers -- ``cli.simulate`` (cli.py:71), ``cli.cmd_bench``
(cli.py:187-191), ``server.Session.run_frame`` (server.py:407),
``oracle.oracle_divergence``, the demos -- run on the GPU while their
``SimState`` stays the reference's numpy dataclass.  Every call uploads the reference state's host arrays into a
device context cached on the state object and downloads the results back into
those same arrays (the e2e host-buffer path).  ``uninstall()`` restores the
originals.
"""

from __future__ import annotations

import sys
import types

import numpy as np

from . import core as _core
from . import frame as _frame
from .collision import pack_colliders as _pack

_SAVED: dict = {}
_ABSENT = object()


def _shadow(ref_state):
    """Device-side SimState mirroring a reference SimState: its x / v / F / C
    mirrors ARE the reference state's arrays (SimState._adopt: uploads read
    them, downloads land in them, no host copies), re-adopted and re-uploaded
    on every call because the caller may have edited them in place."""
    sh = getattr(ref_state, "_b200_shadow", None)
    g = ref_state.grid
    if sh is None or sh.particle_count != len(ref_state.x):
        sh = _core.SimState(_core.Grid(g.resolution, g.extent), ref_state.x, ref_state.v,
                            ref_state.F, ref_state.C, ref_state.mass, ref_state.vol0,
                            ref_state.material_id)
        ref_state._b200_shadow = sh
    else:
        sh.mass, sh.vol0, sh.material_id = ref_state.mass, ref_state.vol0, ref_state.material_id
    for nm in ("x", "v", "F", "C"):
        sh._adopt(nm, getattr(ref_state, nm))
    sh.time = ref_state.time
    sh.step_count = ref_state.step_count
    return sh


def _writeback(ref_state, sh, fields=("x", "v", "F", "C"), grid=True, collision=False):
    newer = tuple(nm for nm in fields if nm in sh._dev_newer)
    if newer:
        sh._download(newer)  # one transfer for all of them
    for nm in fields:
        src = getattr(sh, nm)  # the download (into the adopted array itself when it was adoptable)
        dst = getattr(ref_state, nm)
        if dst is not src:
            np.copyto(dst, src)
    # the shadow's mirrors were only read (into the caller's own arrays): they
    # still equal the device, so the next device call need not upload them
    sh._host_dirty.difference_update(fields)
    d = ref_state.__dict__
    if grid:
        # the dense grid (537 MB at 256^3) is copied back only when read
        d.setdefault("_b200_stale", set()).update(("grid_mv", "grid_m"))
    if collision:
        d.setdefault("_b200_stale", set()).add("_collision")
    ref_state.time = sh.time
    ref_state.step_count = sh.step_count


def _lazy_attr(name):
    """Class-level data descriptor over a reference SimState dataclass field:
    values written by the device path are fetched from the shadow state on
    first read (grid_mv / grid_m downloaded into the caller's own arrays,
    _collision = the merged field of the last substep, core.py:307-309)."""
    def get(self):
        d = self.__dict__
        stale = d.get("_b200_stale")
        if stale and name in stale:
            stale.discard(name)
            sh = d.get("_b200_shadow")
            if name == "_collision":
                d[name] = sh._collision
            else:
                np.copyto(d[name], getattr(sh, name))
        return d.get(name)

    def set(self, value):
        d = self.__dict__
        if d.get("_b200_stale"):
            d["_b200_stale"].discard(name)
        d[name] = value
    return property(get, set)


_MODE = {"deterministic": False}


def _params(p):
    return _core.SimParams(dt=p.dt, substeps_per_frame=p.substeps_per_frame, gravity=tuple(p.gravity),
                           boundary_width=p.boundary_width, boundary=p.boundary,
                           collision_theta=p.collision_theta,
                           accumulation_chunks=p.accumulation_chunks,
                           deterministic=_MODE["deterministic"])


def _mats(materials):
    from .materials import Material
    return [Material(m.young_modulus, m.poisson_ratio, m.density) for m in materials]


def install(softmpm_module, deterministic: bool = False):
    """Patch the reference package in place; returns the module.

    deterministic=True runs every substep in the sorted-order deterministic
    mode (bitwise reproducible, like the reference's fixed-chunk accumulation,
    kernels.py:8-12) instead of the fast atomic mode."""
    core = softmpm_module.core
    _MODE["deterministic"] = bool(deterministic)
    if _SAVED:
        return softmpm_module
    cls = core.SimState
    _SAVED["__lazy__"] = (cls, {a: cls.__dict__.get(a, _ABSENT) for a in ("grid_mv", "grid_m", "_collision")})
    for a in ("grid_mv", "grid_m", "_collision"):
        setattr(cls, a, _lazy_attr(a))

    def p2g(state, materials, params):
        sh = _shadow(state)
        inv = _core.p2g(sh, _mats(materials), _params(params))
        _writeback(state, sh, ("F",))
        return inv

    def grid_update(state, params, collision=None, colliders=None):
        sh = _shadow(state)
        sh.grid_mv = state.grid_mv
        sh.grid_m = state.grid_m
        _core.grid_update(sh, _params(params), collision, _colliders(state, colliders))
        _writeback(state, sh, ())

    def g2p_advect(state, params):
        sh = _shadow(state)
        sh.grid_mv = state.grid_mv
        _core.g2p_advect(sh, _params(params))
        _writeback(state, sh, ("x", "v", "C"), grid=False)

    def substep(state, materials, params, colliders=None):
        sh = _shadow(state)
        inv = _core.substep(sh, _mats(materials), _params(params), _colliders(state, colliders))
        _writeback(state, sh, collision=bool(colliders))
        return inv

    def step(state, materials, params, colliders=None, pose_fn=None):
        sh = _shadow(state)
        rep = _core.step(sh, _mats(materials), _params(params), _colliders(state, colliders),
                         pose_fn)
        _writeback(state, sh, collision=bool(colliders))
        return softmpm_module.core.StepReport(rep.step_index, rep.sim_time, rep.timings_ms,
                                              rep.inverted_particles)

    # §8f consumers: the device splat / marching cubes / metrics, reading the
    # shadow's device-resident particles when the caller's arrays still equal
    # what the last step wrote back (no particle upload per frame)
    surf = getattr(softmpm_module, "surfacing", None)
    scene = getattr(softmpm_module, "scene", None)

    def _ref_mesh(m):
        return surf.SurfaceMesh(vertices=m.vertices, indices=np.asarray(m.indices, dtype=np.int32),
                                uvs=m.uvs, normals=m.normals)

    def splat_density(positions, masses, grid, resolution=None, chunks=8):
        f = _frame.splat_density(positions, masses, _core.Grid(grid.resolution, grid.extent), resolution)
        return surf.ScalarField(values=f.values, dx=f.dx)

    def marching_cubes(fld, iso):
        return _ref_mesh(_frame.marching_cubes(_frame.ScalarField(values=fld.values, dx=fld.dx), iso))

    def extract_surface(state, iso, resolution=None):
        sh = _synced_shadow(state, ("x",))
        return _ref_mesh(_frame.extract_surface(sh, iso, resolution))

    def compute_metrics(state, initial_positions):
        sh = _synced_shadow(state, ("x", "F"))
        m = _frame.compute_metrics(sh, initial_positions)
        return scene.MetricSample(time=state.time, lifted_fraction=m.lifted_fraction,
                                  detached_fraction=m.detached_fraction,
                                  mean_abs_j_minus_1=m.mean_abs_j_minus_1, max_displacement=m.max_displacement)

    new = {"p2g": p2g, "grid_update": grid_update, "g2p_advect": g2p_advect, "substep": substep, "step": step}
    originals = {nm: getattr(core, nm) for nm in new}
    if surf is not None:
        for nm, fn in (("splat_density", splat_density), ("marching_cubes", marching_cubes),
                       ("extract_surface", extract_surface)):
            originals[nm], new[nm] = getattr(surf, nm), fn
    if scene is not None and hasattr(scene, "compute_metrics"):
        originals["compute_metrics"], new["compute_metrics"] = scene.compute_metrics, compute_metrics
    # every binding of the originals in the loaded package -- softmpm.core.step,
    # the softmpm.step re-export, and copies made by `from .core import step`
    # in softmpm.cli / softmpm.server / ... -- is rebound (modules imported
    # later pick up the patched core / surfacing attributes by themselves)
    pkg = softmpm_module.__name__
    mods = {id(softmpm_module): softmpm_module}
    for a in dir(softmpm_module):  # submodules reachable as attributes (also unregistered ones)
        m = getattr(softmpm_module, a, None)
        if isinstance(m, types.ModuleType):
            mods.setdefault(id(m), m)
    for mname, mod in list(sys.modules.items()):
        if mod is not None and (mname == pkg or mname.startswith(pkg + ".")):
            mods.setdefault(id(mod), mod)
    rebound = []
    for mod in mods.values():
        for nm, orig in originals.items():
            if getattr(mod, nm, None) is orig:
                setattr(mod, nm, new[nm])
                rebound.append((mod, nm, orig))
    _SAVED["__rebound__"] = rebound
    return softmpm_module


def _synced_shadow(state, fields):
    """The shadow state with the fields a consumer reads re-adopted (and so
    re-uploaded: the caller may have edited them in place since the last
    installed call; one upload costs less than comparing the arrays)."""
    sh = state.__dict__.get("_b200_shadow")
    if sh is None or len(state.x) != sh.particle_count:
        return _shadow(state)
    for f in fields:
        sh._adopt(f, getattr(state, f))
    return sh


def _colliders(state, colliders):
    # reference RigidCollider objects carry the same fields; they are used as-is
    # (pack_colliders only reads attributes), keeping identity for F7 caching
    return colliders or []


def uninstall(softmpm_module):
    for mod, nm, orig in _SAVED.pop("__rebound__", []):
        setattr(mod, nm, orig)
    cls, attrs = _SAVED.pop("__lazy__", (None, {}))
    for a, orig in attrs.items():
        if orig is _ABSENT:
            delattr(cls, a)
        else:
            setattr(cls, a, orig)  # e.g. the dataclass default _collision = None
    _SAVED.clear()


__all__ = ["install", "uninstall", "_pack"]
