"""CPU checks of the marching-cubes restatement (oracle/mc_oracle.py) against
the reference's own surfacing assertions (tests/test_surfacing.py:41-124 of
the reference: sphere radii, lattice-edge vertices, outward unit normals,
watertight consistent orientation) -- no GPU."""
import numpy as np

from oracle import mc_oracle


def _sphere(n=24, radius=0.3):
    ax = np.arange(n) / n
    x, y, z = np.meshgrid(ax, ax, ax, indexing="ij")
    r = np.sqrt((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2)
    return np.where(r < radius, 1000.0, 0.0), 1.0 / n, radius


def test_oracle_sphere_geometry():
    f, dx, radius = _sphere()
    V, T, N = mc_oracle.marching_cubes(f, 300.0, dx)
    assert len(V) > 100 and len(T) > 100
    r = np.linalg.norm(V - 0.5, axis=1)
    assert np.abs(r - radius).max() < 1.5 * dx
    frac = V / dx
    assert ((np.abs(frac - np.round(frac)) > 1e-9).sum(axis=1) <= 1).all()   # on lattice edges
    assert np.abs(np.linalg.norm(N, axis=1) - 1.0).max() < 1e-12
    assert (np.einsum("ij,ij->i", N, V - 0.5) > 0).all()                    # outward
    v0, v1, v2 = (V[T[:, k]] for k in range(3))
    assert (np.einsum("ij,ij->i", np.cross(v1 - v0, v2 - v0), (v0 + v1 + v2) / 3 - 0.5) > 0).all()
    edges = {(a, b) for t in T for a, b in ((t[0], t[1]), (t[1], t[2]), (t[2], t[0]))}
    assert len(edges) == 3 * len(T) and all((b, a) in edges for a, b in edges)  # watertight


def test_oracle_empty_and_degenerate():
    f, dx, _ = _sphere(n=10)
    V, T, N = mc_oracle.marching_cubes(f, 2000.0, dx)
    assert len(V) == 0 and len(T) == 0
    # an iso level hit exactly at lattice nodes collapses edge vertices onto
    # them: allow_degenerate=False drops the zero-area triangles
    g = np.zeros((6, 6, 6))
    g[2:4, 2:4, 2:4] = 1.0
    V, T, N = mc_oracle.marching_cubes(g, 1.0, 1.0)
    p = V[T]
    assert not ((p[:, 0] == p[:, 1]).all(1) | (p[:, 1] == p[:, 2]).all(1) | (p[:, 0] == p[:, 2]).all(1)).any()
