"""CPU restatement of the reference's isosurface step -- TEST INFRASTRUCTURE ONLY.

The reference triangulates the splatted density with
``skimage.measure.marching_cubes(values, iso, gradient_direction="ascent",
allow_degenerate=False, method="lorensen")`` and scales the lattice-unit
vertices by dx (/root/reference/pkg/src/softmpm/surfacing.py:70-95).
scikit-image is not installable in this image (no index), so its Cython
source and case table cannot be run or read here; this module restates the
published algorithm it implements (Lorensen & Cline 1987, "classic" cases):

  * one vertex on every lattice edge whose end values straddle the iso level
    (inside = value >= iso), at p0 + t (p1 - p0), t = (iso - f0) / (f1 - f0);
  * per-vertex normals from the central-difference gradient of the field
    (one-sided at the lattice boundary) interpolated along the edge with the
    same t, oriented to point out of the dense region (-grad), unit length;
  * per cube, triangles from the 256-case table over the 12 cube edges,
    oriented from inside to outside;
  * allow_degenerate=False: triangles with two coincident vertex positions
    are dropped.

The case table is the one tools/gen_mc_table.py derives (face-consistent
marching-squares pairing, the classic <= 5 triangles per case); skimage's own
table is not available, so triangle-level parity with the reference is
parity with this restatement, while the vertex set and the normals follow
from the algorithm alone.  Vertices are numbered in lattice-edge order
(3 * node + axis, nodes in C order) and triangles are emitted cube by cube in
C order, case-table order within a cube.
"""
from __future__ import annotations

import os
import sys

import numpy as np

_TOOLS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools")
if _TOOLS not in sys.path:
    sys.path.insert(0, _TOOLS)
import gen_mc_table as _T  # noqa: E402

_TABLE = None


def case_table():
    global _TABLE
    if _TABLE is None:
        fs = _T.faces()
        _TABLE = [_T.triangles(c, fs) for c in range(256)]
    return _TABLE


def _gradient(f):
    g = np.empty(f.shape + (3,))
    for a in range(3):
        n = f.shape[a]
        idx = np.arange(n)
        lo = np.maximum(idx - 1, 0)
        hi = np.minimum(idx + 1, n - 1)
        span = (hi - lo).astype(np.float64)
        d = np.take(f, hi, axis=a) - np.take(f, lo, axis=a)
        shape = [1, 1, 1]
        shape[a] = n
        g[..., a] = np.where(span.reshape(shape) > 0, d / np.where(span > 0, span, 1.0).reshape(shape), 0.0)
    return g


def marching_cubes(values, iso: float, dx: float):
    """(vertices (V, 3) metres, triangles (T, 3) int32, normals (V, 3)) of the
    iso surface of a nodal field; empty arrays when it is never crossed."""
    f = np.asarray(values, dtype=np.float64)
    nx, ny, nz = f.shape
    inside = f >= iso
    grad = _gradient(f)
    vid = -np.ones(f.shape + (3,), dtype=np.int64)
    verts, norms = [], []
    # lattice edges in (node, axis) order
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                for axis in range(3):
                    i2, j2, k2 = i + (axis == 0), j + (axis == 1), k + (axis == 2)
                    if i2 >= nx or j2 >= ny or k2 >= nz or inside[i, j, k] == inside[i2, j2, k2]:
                        continue
                    f0, f1 = f[i, j, k], f[i2, j2, k2]
                    t = (iso - f0) / (f1 - f0)
                    p0 = np.array([i, j, k], dtype=np.float64)
                    p1 = np.array([i2, j2, k2], dtype=np.float64)
                    g = -(grad[i, j, k] + t * (grad[i2, j2, k2] - grad[i, j, k]))
                    nrm = np.sqrt(np.dot(g, g))
                    vid[i, j, k, axis] = len(verts)
                    verts.append((p0 + t * (p1 - p0)) * dx)
                    norms.append(g / nrm if nrm > 1e-30 else np.zeros(3))
    if not verts:
        return np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros((0, 3))
    table = case_table()
    corners = _T.CORNERS.astype(int)
    tris = []
    for i in range(nx - 1):
        for j in range(ny - 1):
            for k in range(nz - 1):
                case = 0
                for q in range(8):
                    di, dj, dk = corners[q]
                    case |= int(inside[i + di, j + dj, k + dk]) << q
                for tri in table[case]:
                    ids = []
                    for e in tri:
                        a, b = _T.EDGES[e]
                        ca, cb = corners[a], corners[b]
                        lo = np.minimum(ca, cb)
                        axis = int(np.nonzero(ca != cb)[0][0])
                        ids.append(vid[i + lo[0], j + lo[1], k + lo[2], axis])
                    tris.append(ids)
    V = np.array(verts)
    T = np.array(tris, dtype=np.int64).reshape(-1, 3)
    # allow_degenerate=False
    p = V[T]
    keep = ~((p[:, 0] == p[:, 1]).all(1) | (p[:, 1] == p[:, 2]).all(1) | (p[:, 0] == p[:, 2]).all(1))
    return V, T[keep].astype(np.int32), np.array(norms)
