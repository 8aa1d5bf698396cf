"""MPMF frame wire format of the interactive session host (server.py:36-124):
a little-endian, padding-free binary frame carrying the surface mesh and the
tool poses.

`encode_frame` / `decode_frame` keep the reference's host codec (same bytes);
`encode_surface_frame` is the device path: splat -> marching cubes -> the
frame body packed by a kernel from the device mesh (f32 vertices, normals,
planar UVs, u32 indices) and read back once, so the particles and the fp64
mesh never cross PCIe."""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ParameterError, SimError

MAGIC = b"MPMF"
HEADER = struct.Struct("<4sIfII")          # magic, frame index, sim time, vertex count, triangle count
COLLIDER_REC = struct.Struct("<I3f4fB")    # id, translation, quaternion (x, y, z, w), jaw closed
MAX_VERTICES = 1 << 24


class FrameTooLarge(SimError):
    """Mesh exceeds the wire format's vertex budget; the frame is skipped."""


@dataclass
class ColliderPose:
    id: int
    translation: np.ndarray
    quaternion: np.ndarray  # (x, y, z, w)
    jaw_closed: bool


@dataclass
class DecodedFrame:
    frame_index: int
    sim_time: float
    vertices: np.ndarray
    normals: np.ndarray
    uvs: np.ndarray
    indices: np.ndarray
    colliders: list[ColliderPose]


def _collider_block(colliders) -> bytes:
    out = [struct.pack("<I", len(colliders))]
    for c in colliders:
        t = np.asarray(c.translation, dtype=float)
        q = np.asarray(c.quaternion, dtype=float)
        out.append(COLLIDER_REC.pack(int(c.id), *t, *q, 1 if c.jaw_closed else 0))
    return b"".join(out)


def encode_frame(mesh, colliders: list[ColliderPose], frame_index: int, sim_time: float) -> bytes:
    """Serialize one frame (server.py:65-92): header + 32 V + 12 T + 4 + 33 C
    bytes; FrameTooLarge above MAX_VERTICES vertices."""
    v = np.ascontiguousarray(mesh.vertices, dtype="<f4")
    nv = len(v)
    if nv > MAX_VERTICES:
        raise FrameTooLarge(f"{nv} vertices exceeds the {MAX_VERTICES} cap")
    normals = mesh.normals if mesh.normals is not None else np.zeros((nv, 3))
    uvs = mesh.uvs if mesh.uvs is not None else np.zeros((nv, 2))
    tris = np.ascontiguousarray(mesh.indices, dtype="<u4")
    return b"".join([HEADER.pack(MAGIC, frame_index, sim_time, nv, len(tris)), v.tobytes(),
                     np.ascontiguousarray(normals, dtype="<f4").tobytes(),
                     np.ascontiguousarray(uvs, dtype="<f4").tobytes(), tris.tobytes(), _collider_block(colliders)])


def decode_frame(data: bytes) -> DecodedFrame:
    """Exact inverse of encode_frame (server.py:95-124)."""
    magic, frame_index, sim_time, nv, nt = HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise SimError("bad frame magic")
    off = HEADER.size

    def take(count, dtype, cols):
        nonlocal off
        arr = np.frombuffer(data, dtype=dtype, count=count * cols, offset=off)
        off += arr.nbytes
        return arr.reshape(count, cols)

    vertices, normals, uvs, indices = take(nv, "<f4", 3), take(nv, "<f4", 3), take(nv, "<f4", 2), take(nt, "<u4", 3)
    (ncol,) = struct.unpack_from("<I", data, off)
    off += 4
    colliders = []
    for _ in range(ncol):
        rec = COLLIDER_REC.unpack_from(data, off)
        off += COLLIDER_REC.size
        colliders.append(ColliderPose(id=rec[0], translation=np.array(rec[1:4]), quaternion=np.array(rec[4:8]),
                                      jaw_closed=bool(rec[8])))
    if off != len(data):
        raise SimError(f"frame has {len(data) - off} trailing bytes")
    return DecodedFrame(frame_index, sim_time, vertices, normals, uvs, indices, colliders)


def encode_surface_frame(state, iso: float, colliders: list[ColliderPose], frame_index: int, sim_time: float,
                         resolution=None) -> bytes:
    """encode_frame(extract_surface(state, iso, resolution), ...) with the
    surface built and packed on the device: the same bytes, one readback of
    the frame body."""
    from .frame import _device_state, _field_geometry
    if iso <= 0.0:
        raise ParameterError("iso level must be positive")
    tail = _collider_block(colliders)
    if state.particle_count == 0:
        return HEADER.pack(MAGIC, frame_index, sim_time, 0, 0) + tail
    res, dx = _field_geometry(state.grid, resolution)
    ctx = _device_state(state)
    r = (ctypes.c_int32 * 3)(*res)
    ctx.call("mpm_splat_density", _lib.ptr(None), _lib.ptr(None), ctypes.c_int64(0), r, ctypes.c_double(dx),
             _lib.ptr(None))
    nv, nt = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("mpm_marching_cubes", _lib.ptr(None), _lib.ptr(None, _lib._I32), ctypes.c_double(dx),
             ctypes.c_double(iso), ctypes.byref(nv), ctypes.byref(nt))
    if nv.value > MAX_VERTICES:
        raise FrameTooLarge(f"{nv.value} vertices exceeds the {MAX_VERTICES} cap")
    body = 32 * nv.value + 12 * nt.value
    buf = bytearray(HEADER.size + body + len(tail))
    HEADER.pack_into(buf, 0, MAGIC, frame_index, sim_time, nv.value, nt.value)
    ext = np.ascontiguousarray(state.grid.extent, dtype=np.float64)
    n = ctypes.c_int64(0)
    if body:
        view = (ctypes.c_uint8 * body).from_buffer(buf, HEADER.size)
        ctx.call("mpm_mesh_encode", _lib.ptr(ext), ctypes.cast(view, ctypes.c_void_p), ctypes.c_int64(body),
                 ctypes.byref(n))
        del view
    buf[HEADER.size + body:] = tail
    return bytes(buf)
