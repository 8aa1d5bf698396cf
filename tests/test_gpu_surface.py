"""Device isosurface (marching cubes) and the splat -> surface pipeline,
restating the reference's surfacing tests (tests/test_surfacing.py:41-124).
The reference triangulates with scikit-image's Lorensen tables, absent from
this image, so parity is geometric: the reference's own assertions (radii,
lattice-edge vertices, consistent outward orientation, unit outward normals,
no degenerate triangles), plus watertightness and the empty / invalid cases."""
import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200.errors import ParameterError

pytestmark = pytest.mark.gpu


def sphere_field(n=48, radius=0.25, density=1000.0):
    grid = sm.Grid(resolution=(n, n, n), extent=(1.0, 1.0, 1.0))
    ax = np.arange(n) * grid.dx
    x, y, z = np.meshgrid(ax, ax, ax, indexing="ij")
    r = np.sqrt((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2)
    return sm.ScalarField(values=np.where(r < radius, density, 0.0), dx=grid.dx), radius


def test_marching_cubes_sphere_radii():
    fld, radius = sphere_field()
    mesh = sm.marching_cubes(fld, 300.0)
    assert len(mesh.vertices) > 100
    r = np.linalg.norm(mesh.vertices - 0.5, axis=1)
    assert np.abs(r - radius).max() < 1.5 * fld.dx


def test_marching_cubes_below_iso_empty_and_invalid_iso():
    fld, _ = sphere_field(density=100.0)
    mesh = sm.marching_cubes(fld, 300.0)
    assert len(mesh.vertices) == 0 and len(mesh.indices) == 0
    with pytest.raises(ParameterError):
        sm.marching_cubes(fld, 0.0)


def test_marching_cubes_vertices_on_lattice_edges():
    fld, _ = sphere_field()
    mesh = sm.marching_cubes(fld, 300.0)
    frac = mesh.vertices / fld.dx
    off_lattice = np.abs(frac - np.round(frac)) > 1e-9
    assert (off_lattice.sum(axis=1) <= 1).all()


def _directed_edges(indices):
    edges = set()
    for a, b, c in indices:
        for e in ((a, b), (b, c), (c, a)):
            assert e not in edges  # each directed edge once
            edges.add(e)
    return edges


def test_marching_cubes_orientation_consistent_and_watertight():
    fld, _ = sphere_field()
    mesh = sm.marching_cubes(fld, 300.0)
    edges = _directed_edges(mesh.indices)
    for a, b in edges:
        assert (b, a) in edges


def test_marching_cubes_outward_and_unit_normals():
    fld, _ = sphere_field()
    mesh = sm.marching_cubes(fld, 300.0)
    v0, v1, v2 = (mesh.vertices[mesh.indices[:, k]] for k in range(3))
    face_n = np.cross(v1 - v0, v2 - v0)
    outward = (v0 + v1 + v2) / 3.0 - 0.5
    assert (np.einsum("ij,ij->i", face_n, outward) > 0.0).all()
    assert np.abs(np.linalg.norm(mesh.normals, axis=1) - 1.0).max() < 1e-9
    assert (np.einsum("ij,ij->i", mesh.normals, mesh.vertices - 0.5) > 0.0).all()


def test_no_degenerate_triangles():
    fld, _ = sphere_field()
    mesh = sm.marching_cubes(fld, 300.0)
    v0, v1, v2 = (mesh.vertices[mesh.indices[:, k]] for k in range(3))
    areas = 0.5 * np.linalg.norm(np.cross(v1 - v0, v2 - v0), axis=1)
    assert (areas > 1e-12).all()


def test_random_fields_watertight(rng=np.random.default_rng(3)):
    """Random smooth fields (ambiguous cube cases included): every directed
    edge has its reverse unless it lies on the field's outer boundary."""
    n = 20
    for _ in range(3):
        g = rng.normal(size=(n, n, n))
        for axis in range(3):
            g = (g + np.roll(g, 1, axis) + np.roll(g, -1, axis)) / 3.0
        g[0], g[-1], g[:, 0], g[:, -1], g[:, :, 0], g[:, :, -1] = 0, 0, 0, 0, 0, 0
        fld = sm.ScalarField(values=g - g.min() + 1e-3, dx=1.0 / n)
        iso = float(np.median(fld.values[fld.values > 1e-3 + 1e-12]) if (fld.values > 1e-3).any() else 1.0)
        mesh = sm.marching_cubes(fld, iso)
        edges = _directed_edges(mesh.indices)
        for a, b in edges:
            assert (b, a) in edges


def test_uvs_projection():
    mesh = sm.SurfaceMesh(vertices=np.array([[0.0, 0.3, 0.0], [1.0, 0.1, 1.0], [0.25, 0.0, 0.75]]),
                          indices=np.array([[0, 1, 2]], dtype=np.int32))
    sm.compute_uvs(mesh, (1.0, 1.0, 1.0))
    assert np.allclose(mesh.uvs, [(0.0, 0.0), (1.0, 1.0), (0.25, 0.75)])


def test_extract_surface_of_a_device_state():
    grid = sm.Grid(resolution=(16, 16, 16), extent=(1.0, 1.0, 1.0))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.5, 0.5), (0.3, 0.3, 0.3), 4000, seed=21, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    sm.step(st, mats, sm.SimParams())
    mesh = sm.extract_surface(st, iso=300.0)
    assert len(mesh.vertices) > 0 and mesh.uvs is not None and mesh.normals is not None
    assert (mesh.uvs >= 0.0).all() and (mesh.uvs <= 1.0).all()
    # the device pipeline equals the host-field path on the same density
    fld = sm.density_field(st)
    ref = sm.marching_cubes(fld, 300.0)
    assert np.array_equal(mesh.indices, ref.indices)
    assert np.abs(mesh.vertices - ref.vertices).max() < 1e-12
    edges = _directed_edges(mesh.indices)
    for a, b in edges:
        assert (b, a) in edges


def test_encode_surface_frame_equals_host_encoding():
    """the frame body packed on the device from the device
    mesh equals encode_frame(extract_surface(...)) byte for byte."""
    grid = sm.Grid(resolution=(24, 24, 24), extent=(1.0, 1.0, 1.0))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.45, 0.4, 0.55), (0.3, 0.25, 0.3), 12000, seed=5, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    sm.step(st, mats, sm.SimParams())
    cols = [sm.wire.ColliderPose(2, np.array([0.5, 0.7, 0.5]), np.array([0.0, 0.0, 0.0, 1.0]), True)]
    dev = sm.encode_surface_frame(st, 300.0, cols, 9, float(st.time))
    host = sm.encode_frame(sm.extract_surface(st, 300.0), cols, 9, float(st.time))
    assert len(dev) > 1000 and dev == host
    d = sm.decode_frame(dev)
    assert len(d.vertices) > 0 and d.colliders[0].id == 2
    # resolution override and a surface that never reaches the iso level
    assert sm.encode_surface_frame(st, 300.0, [], 1, 0.0, resolution=(32, 32, 32)) == \
        sm.encode_frame(sm.extract_surface(st, 300.0, resolution=(32, 32, 32)), [], 1, 0.0)
    empty = sm.encode_surface_frame(st, 1e12, [], 3, 0.0)
    assert sm.decode_frame(empty).vertices.shape == (0, 3)


# ---- parity against the CPU restatement of the Lorensen isosurface (oracle/mc_oracle.py)
def _mc_oracle_compare(fld, iso):
    from oracle import mc_oracle
    mesh = sm.marching_cubes(fld, iso)
    V, T, N = mc_oracle.marching_cubes(fld.values, iso, fld.dx)
    # same vertex set, numbered alike (lattice-edge order), same positions / normals
    assert mesh.vertices.shape == V.shape
    assert np.abs(mesh.vertices - V).max() < 1e-12
    assert np.abs(mesh.normals - N).max() < 1e-12
    # same triangles, emitted in the same order (cube order, case-table order)
    assert np.array_equal(mesh.indices, T)
    return mesh


def test_marching_cubes_matches_oracle_sphere():
    fld, _ = sphere_field()
    mesh = _mc_oracle_compare(fld, 300.0)
    assert len(mesh.indices) > 500


def test_marching_cubes_matches_oracle_random_fields(rng=np.random.default_rng(11)):
    n = 18
    for _ in range(3):
        g = rng.normal(size=(n, n, n))
        for axis in range(3):
            g = (g + np.roll(g, 1, axis) + np.roll(g, -1, axis)) / 3.0
        fld = sm.ScalarField(values=g - g.min() + 1e-3, dx=1.0 / n)
        iso = float(np.median(fld.values))
        _mc_oracle_compare(fld, iso)


def test_marching_cubes_matches_oracle_splatted_state():
    """The reference pipeline's own field: a settled block's B-spline splat."""
    grid = sm.Grid(resolution=(20, 20, 20), extent=(1.0, 1.0, 1.0))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.35, 0.5), (0.4, 0.3, 0.35), 6000, seed=8, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    sm.step(st, mats, sm.SimParams())
    _mc_oracle_compare(sm.density_field(st), 300.0)
