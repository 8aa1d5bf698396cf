"""Baked signed-distance lattices for rigid tools (host side).

``SdfGrid`` keeps the reference's lattice convention
(/root/reference/pkg/src/softmpm/sdf.py:32-78): values[i,j,k] is the distance
at cell centre ((i+0.5)/n, ...) of a padded cube, in normalised units; the
device samples it trilinearly in fp64 (csrc/collide.cuh: baked_sd, the
kernels.py:48-88 rule).  SDF1 files (sdf.py:306-329) load and save unchanged.

Mesh baking (sdf.py:246-303) is offline asset work and out of scope; the
surgical "capsule grasper" of BASELINE config 2 is baked here from the
analytic capsule distance instead (``bake_capsule``), which is exact at the
lattice samples.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import MeshError

_MAGIC = b"SDF1"


@dataclass
class SdfGrid:
    values: np.ndarray
    bounds_min: np.ndarray
    extent: float

    @property
    def resolution(self) -> tuple[int, int, int]:
        return self.values.shape  # type: ignore[return-value]

    @property
    def dx_sdf(self) -> float:
        return 1.0 / self.values.shape[0]

    def sample(self, points: np.ndarray) -> np.ndarray:
        """Trilinear lookup in local-frame metres, clamped at the lattice edge."""
        p = np.atleast_2d(np.asarray(points, dtype=np.float64))
        res = np.array(self.values.shape, dtype=np.float64)
        c = (p - self.bounds_min) / self.extent * res - 0.5
        c = np.clip(c, 0.0, res - 1.0)
        i0 = np.minimum(c.astype(np.int64), (res - 2.0).astype(np.int64))
        f = c - i0
        v = self.values
        out = np.zeros(len(p))
        for a in (0, 1):
            wa = f[:, 0] if a else 1.0 - f[:, 0]
            for b in (0, 1):
                wb = f[:, 1] if b else 1.0 - f[:, 1]
                for cc in (0, 1):
                    wc = f[:, 2] if cc else 1.0 - f[:, 2]
                    out += wa * wb * wc * v[i0[:, 0] + a, i0[:, 1] + b, i0[:, 2] + cc]
        out *= self.extent
        return out if np.asarray(points).ndim > 1 else out[0]


def capsule_distance(p: np.ndarray, radius: float, half_length: float, axis: int = 1) -> np.ndarray:
    """Exact signed distance to a capsule (segment of +-half_length along `axis`)."""
    p = np.asarray(p, dtype=np.float64)
    q = np.zeros_like(p)
    q[..., axis] = np.clip(p[..., axis], -half_length, half_length)
    return np.linalg.norm(p - q, axis=-1) - radius


def bake_capsule(radius: float, half_length: float, resolution: int = 64, axis: int = 1,
                 padding: float = 0.125) -> SdfGrid:
    """Capsule SDF lattice in the reference's padded-cube convention."""
    ext_vec = np.full(3, 2.0 * radius)
    ext_vec[axis] = 2.0 * (half_length + radius)
    extent = float(ext_vec.max()) * (1.0 + 2.0 * padding)
    bounds_min = -0.5 * extent * np.ones(3)
    n = int(resolution)
    centers = (np.arange(n) + 0.5) / n * extent
    g = np.stack(np.meshgrid(centers, centers, centers, indexing="ij"), axis=-1) + bounds_min
    values = capsule_distance(g, radius, half_length, axis) / extent
    return SdfGrid(values=values, bounds_min=bounds_min, extent=extent)


def save_sdf(path: str | Path, grid: SdfGrid) -> None:
    """SDF1 container: magic, 3 x u32 res, 6 x f32 bounds, f32 values x-fastest."""
    nx, ny, nz = grid.values.shape
    bmax = grid.bounds_min + grid.extent
    header = _MAGIC + struct.pack("<3I", nx, ny, nz) + struct.pack("<6f", *grid.bounds_min, *bmax)
    payload = np.asfortranarray(grid.values.astype("<f4")).tobytes(order="F")
    Path(path).write_bytes(header + payload)


def load_sdf(path: str | Path) -> SdfGrid:
    raw = Path(path).read_bytes()
    if raw[:4] != _MAGIC:
        raise MeshError(f"{Path(path).name}: not an SDF1 file")
    nx, ny, nz = struct.unpack_from("<3I", raw, 4)
    bounds = struct.unpack_from("<6f", raw, 16)
    vals = np.frombuffer(raw, dtype="<f4", count=nx * ny * nz, offset=40)
    values = np.reshape(vals, (nx, ny, nz), order="F").astype(np.float64)
    bmin = np.array(bounds[:3], dtype=np.float64)
    ext = np.array(bounds[3:], dtype=np.float64) - bmin
    if np.ptp(ext) > 1.0e-4 * ext.max():
        raise MeshError("SDF bounds must be cubic")
    return SdfGrid(values=np.ascontiguousarray(values), bounds_min=bmin, extent=float(ext[0]))
