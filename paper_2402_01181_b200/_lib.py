"""ctypes binding of libsoftmpm_b200.so (include/softmpm_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every entry point raises.  ``build()`` compiles the library
in-tree with nvcc for sm_100a (csrc/Makefile).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .errors import ParameterError, SimError, StencilError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SOFTMPM_LIB") or os.path.join(_HERE, "libsoftmpm_b200.so")
_lib = None

MPM_OK, MPM_EINVAL, MPM_ENOMEM, MPM_ECUDA, MPM_ESTATE, MPM_ESTENCIL = 0, -1, -2, -3, -4, -5
FIELD_X, FIELD_V, FIELD_F, FIELD_C = 1, 2, 4, 8
FIELD_ALL = 15
DOWNLOAD_KEEP_EQUAL = 16  # MPM_DOWNLOAD_KEEP_EQUAL

_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)
_VP = ctypes.c_void_p

EXPORTS = (
    "mpm_create", "mpm_destroy", "mpm_set_config", "mpm_last_error", "mpm_version",
    "mpm_set_materials", "mpm_upload_particles", "mpm_upload_fields", "mpm_download_particles",
    "mpm_particle_count", "mpm_upload_grid", "mpm_download_grid", "mpm_set_colliders",
    "mpm_set_pose_table", "mpm_p2g", "mpm_grid_update", "mpm_g2p", "mpm_substeps",
    "mpm_collision_field", "mpm_has_nan", "mpm_launch_count", "mpm_host_alloc", "mpm_host_free",
    "mpm_set_timing", "mpm_get_timing", "mpm_set_option", "mpm_set_slab", "mpm_halo_buffers",
    "mpm_stage_begin", "mpm_stage_particles", "mpm_stage_grid", "mpm_stage_end", "mpm_halo_pack",
    "mpm_halo_unpack_add", "mpm_halo_pack_vel", "mpm_halo_unpack_vel", "mpm_extract_migrants",
    "mpm_append_particles", "mpm_reserve", "mpm_download_ids", "mpm_device_copy", "mpm_set_ids",
    "mpm_download_rows", "mpm_metrics", "mpm_splat_density", "mpm_splat_density_host",
    "mpm_marching_cubes", "mpm_mesh_fetch", "mpm_mesh_encode", "mpm_ipc_blob_size", "mpm_ipc_export", "mpm_ipc_import", "mpm_ipc_mode",
    "mpm_ipc_halo", "mpm_get_stat", "mpm_peer_connect",
)


class MpmConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("res", ctypes.c_int * 3), ("dx", ctypes.c_double),
                ("dt", ctypes.c_double), ("gravity", ctypes.c_double * 3),
                ("boundary_width", ctypes.c_int), ("stick", ctypes.c_int),
                ("theta", ctypes.c_double), ("stress_form", ctypes.c_int),
                ("mode_live", ctypes.c_int), ("deterministic", ctypes.c_int),
                ("rebin_interval", ctypes.c_int), ("env_tiles", ctypes.c_int * 3),
                ("colliders_per_env", ctypes.c_int)]


def build(force: bool = False) -> str:
    """Compile csrc/ into libsoftmpm_b200.so (nvcc, sm_100a)."""
    cmd = ["make", "-C", os.path.join(_HERE, "csrc")]
    if force:
        cmd.append("-B")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SimError(f"CUDA extension {LIB_PATH} is not built; run `python __graft_entry__.py`"
                       " (build()) -- there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    L.mpm_create.argtypes = [ctypes.POINTER(_VP), ctypes.POINTER(MpmConfig)]
    L.mpm_destroy.argtypes = [_VP]
    L.mpm_set_config.argtypes = [_VP, ctypes.POINTER(MpmConfig)]
    L.mpm_last_error.argtypes = [_VP]
    L.mpm_last_error.restype = ctypes.c_char_p
    L.mpm_version.restype = ctypes.c_char_p
    L.mpm_set_materials.argtypes = [_VP, _D, _D, ctypes.c_int]
    L.mpm_upload_particles.argtypes = [_VP, ctypes.c_int64, _D, _D, _D, _D, _D, _D, _I32]
    L.mpm_upload_fields.argtypes = [_VP, ctypes.c_uint32, _D, _D, _D, _D]
    L.mpm_download_particles.argtypes = [_VP, ctypes.c_uint32, _D, _D, _D, _D]
    L.mpm_particle_count.argtypes = [_VP]
    L.mpm_particle_count.restype = ctypes.c_int64
    L.mpm_upload_grid.argtypes = [_VP, ctypes.c_int, _D, _D]
    L.mpm_download_grid.argtypes = [_VP, _D, _D]
    L.mpm_set_colliders.argtypes = [_VP, ctypes.c_int, _I32, _D, _D, _D, _D, _D, _D, _I32, _D,
                                    ctypes.c_int64, _I64, _I32, _D, _D]
    L.mpm_set_pose_table.argtypes = [_VP, ctypes.c_int, _D, _D, _D, _D, _I32]
    L.mpm_p2g.argtypes = [_VP, _I64]
    L.mpm_grid_update.argtypes = [_VP, ctypes.c_int]
    L.mpm_g2p.argtypes = [_VP]
    L.mpm_substeps.argtypes = [_VP, ctypes.c_int, ctypes.c_int, _I64, _D]
    L.mpm_collision_field.argtypes = [_VP, ctypes.c_double, _D, _I32]
    L.mpm_has_nan.argtypes = [_VP, ctypes.POINTER(ctypes.c_int)]
    L.mpm_launch_count.argtypes = [_VP]
    L.mpm_launch_count.restype = ctypes.c_int64
    L.mpm_host_alloc.argtypes = [ctypes.c_int64]
    L.mpm_host_alloc.restype = _VP
    L.mpm_host_free.argtypes = [_VP]
    L.mpm_set_timing.argtypes = [_VP, ctypes.c_int]
    L.mpm_get_timing.argtypes = [_VP, _D]
    L.mpm_set_option.argtypes = [_VP, ctypes.c_char_p, ctypes.c_int]
    L.mpm_get_stat.argtypes = [_VP, ctypes.c_int, _I64]
    L.mpm_peer_connect.argtypes = [_VP, ctypes.c_int, _VP]
    _IP = ctypes.POINTER(ctypes.c_int)
    _PP = ctypes.POINTER(_VP)
    L.mpm_set_slab.argtypes = [_VP, _IP, _IP, ctypes.c_int]
    L.mpm_halo_buffers.argtypes = [_VP, ctypes.c_int, _PP, _PP, _PP, _PP, _I64]
    L.mpm_stage_begin.argtypes = [_VP, ctypes.c_int, ctypes.c_int]
    L.mpm_stage_particles.argtypes = [_VP, ctypes.c_int]
    L.mpm_stage_grid.argtypes = [_VP, ctypes.c_int, ctypes.c_int]
    L.mpm_stage_end.argtypes = [_VP, _I64]
    L.mpm_halo_pack.argtypes = [_VP, ctypes.c_int, _I64]
    L.mpm_halo_unpack_add.argtypes = [_VP, ctypes.c_int, ctypes.c_int64]
    L.mpm_halo_pack_vel.argtypes = [_VP, ctypes.c_int, _I64]
    L.mpm_halo_unpack_vel.argtypes = [_VP, ctypes.c_int, ctypes.c_int64]
    L.mpm_extract_migrants.argtypes = [_VP, ctypes.c_int, ctypes.c_int, _I64, _I64, _PP, _PP, _I64]
    L.mpm_append_particles.argtypes = [_VP, _VP, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
    L.mpm_reserve.argtypes = [_VP, ctypes.c_int64]
    L.mpm_download_ids.argtypes = [_VP, _I32, _D]
    L.mpm_device_copy.argtypes = [_VP, _VP, ctypes.c_int64]
    L.mpm_set_ids.argtypes = [_VP, _I32]
    L.mpm_download_rows.argtypes = [_VP, _I32, _D, _D, _D, _D]
    L.mpm_metrics.argtypes = [_VP, _D, ctypes.c_double, _D]
    L.mpm_splat_density.argtypes = [_VP, _D, _D, ctypes.c_int64, _I32, ctypes.c_double, _D]
    L.mpm_splat_density_host.argtypes = [ctypes.c_int, _D, _D, ctypes.c_int64, _I32, ctypes.c_double, _D]
    L.mpm_marching_cubes.argtypes = [_VP, _D, _I32, ctypes.c_double, ctypes.c_double, _I64, _I64]
    L.mpm_mesh_fetch.argtypes = [_VP, _D, _I32, _D]
    L.mpm_mesh_encode.argtypes = [_VP, _D, _VP, ctypes.c_int64, _I64]
    L.mpm_ipc_blob_size.restype = ctypes.c_int64
    L.mpm_ipc_export.argtypes = [_VP, ctypes.c_int, ctypes.c_char_p]
    L.mpm_ipc_import.argtypes = [_VP, ctypes.c_int, ctypes.c_char_p]
    L.mpm_ipc_halo.argtypes = [_VP, ctypes.c_int, ctypes.c_int]
    L.mpm_ipc_mode.argtypes = [_VP, ctypes.POINTER(ctypes.c_int)]
    _lib = L
    return L


def ptr(a: np.ndarray | None, kind=_D):
    if a is None:
        return ctypes.cast(None, kind)
    return a.ctypes.data_as(kind)


def check(rc: int, handle=None, what: str = "") -> None:
    if rc == MPM_OK:
        return
    msg = ""
    if handle is not None:
        raw = lib().mpm_last_error(handle)
        msg = raw.decode() if raw else ""
    text = f"{what}: {msg or 'error code ' + str(rc)}"
    if rc == MPM_EINVAL:
        raise ParameterError(text)
    if rc == MPM_ESTENCIL:
        raise StencilError(text)
    raise SimError(text)


class Context:
    """Owning handle of one device-side simulation context (one SimState)."""

    def __init__(self, cfg: MpmConfig):
        L = lib()
        h = _VP()
        rc = L.mpm_create(ctypes.byref(h), ctypes.byref(cfg))
        if rc == MPM_ECUDA:
            raise SimError("mpm_create: no usable CUDA device (sm_100a build, no CPU fallback)")
        check(rc, None, "mpm_create")
        self.h = h
        self.cfg = cfg

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.mpm_destroy(h)
            self.h = None

    def call(self, name: str, *args) -> None:
        check(getattr(lib(), name)(self.h, *args), self.h, name)

    @property
    def launches(self) -> int:
        return int(lib().mpm_launch_count(self.h))
