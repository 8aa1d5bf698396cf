"""Generate the golden fixtures in tests/golden/ from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports softmpm from /root/reference/pkg/src (with a scikit-image stub,
surfacing.py is off the hot path) and records inputs and outputs of
the reference's own hot-path entry points:

  * substep_colliders.npz -- core.substep (kernels.py numba path, kernel
    stress form, 8 chunks) with a rotated moving Box (Coulomb) and a Baked SDF
    (sticky) collider: state after 1 and 10 substeps, grid + collision field
    after the first substep.
  * floor_block.npz -- a 2000-particle Neo-Hookean block in the floor band
    (stress path exercised, SURVEY §8d C1 note): x/v/F/C after 1, 10, 100
    substeps with no colliders.
  * spec_reference.npz -- reference.reference_substep (F^-T loop-nest
    oracle, reference.py:14-200): state after 5 substeps.
  * stage_ops.npz -- p2g / grid_update / g2p_advect stage outputs on a
    random state (conftest.random_state-like).
  * kinematics.npz -- scene.pose_at on a rotating keyframe trajectory and
    sampling.sample_box positions for a fixed seed.
  * frame_ops.npz -- surfacing.splat_density on the test_surfacing blob
    (sim lattice and a 2x finer one) and scene.compute_metrics on a block
    after 40 substeps (the frame consumers of SURVEY §8f).
"""
import os
import sys
import types

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sk = types.ModuleType("skimage")
sk.measure = types.ModuleType("skimage.measure")
sys.modules.setdefault("skimage", sk)
sys.modules.setdefault("skimage.measure", sk.measure)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from scipy.spatial.transform import Rotation  # noqa: E402

import softmpm as sm  # noqa: E402
from softmpm.meshio import box_mesh  # noqa: E402
from softmpm.reference import reference_substep  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def state_arrays(st, prefix):
    return {f"{prefix}_x": st.x.copy(), f"{prefix}_v": st.v.copy(),
            f"{prefix}_F": st.F.copy(), f"{prefix}_C": st.C.copy()}


def packed_arrays(p, prefix="col"):
    keys = ["kind", "half", "rotation", "translation", "linear_velocity", "angular_velocity",
            "friction", "mode", "sdf_values", "sdf_offset", "sdf_resolution",
            "sdf_bounds_min", "sdf_extent"]
    return {f"{prefix}_{k}": np.asarray(getattr(p, k)).copy() for k in keys}


def substep_colliders():
    rng = np.random.default_rng(7)
    grid = sm.Grid(resolution=(24, 20, 28), extent=(1.0, 20 / 24, 28 / 24))
    mats = [sm.Material(1e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.16, 0.45), (0.3, 0.15, 0.3), 1200, seed=3, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    st.v[:] = rng.normal(0, 0.3, st.v.shape)
    st.C[:] = rng.normal(0, 1.0, st.C.shape)
    st.F[:] = np.eye(3) + rng.normal(0, 0.05, st.F.shape)
    verts, tris = box_mesh(size=(0.2, 0.1, 0.2))
    baked = sm.bake_sdf(verts, tris, resolution=24)
    cols = [sm.RigidCollider(id=0, shape=sm.Box(np.array([0.1, 0.03, 0.1])),
                             translation=np.array([0.5, 0.26, 0.45]),
                             rotation=Rotation.from_euler("z", 20, degrees=True).as_matrix(),
                             linear_velocity=np.array([0, -0.5, 0]),
                             angular_velocity=np.array([0, 0, 0.3]), friction_mu=0.4),
            sm.RigidCollider(id=1, shape=sm.Baked(baked), translation=np.array([0.3, 0.22, 0.45]),
                             friction_mu=0.2, mode="sticky")]
    params = sm.SimParams()
    out = {"res": np.array(grid.resolution), "extent": np.array(grid.extent),
           "E": 1e4, "nu": 0.3, "rho": 1000.0, "mass": st.mass.copy(), "vol0": st.vol0.copy()}
    out.update(state_arrays(st, "in"))
    inv = sm.substep(st, mats, params, cols)
    out.update(packed_arrays(st._packed))
    out.update(state_arrays(st, "s1"))
    out["s1_inverted"] = inv
    out["s1_grid_mv"] = st.grid_mv.copy()
    out["s1_grid_m"] = st.grid_m.copy()
    out["s1_dist"] = st._collision.distance.copy()
    out["s1_obj"] = st._collision.object_id.copy()
    for _ in range(9):
        sm.substep(st, mats, params, cols)
    out.update(state_arrays(st, "s10"))
    np.savez_compressed(os.path.join(OUT, "substep_colliders.npz"), **out)


def floor_block():
    grid = sm.Grid(resolution=(32, 32, 32))
    mats = [sm.Material(1e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.14, 0.5), (0.3, 0.16, 0.3), 2000, seed=1, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    params = sm.SimParams()
    out = {"res": np.array(grid.resolution), "extent": np.array(grid.extent),
           "E": 1e4, "nu": 0.3, "rho": 1000.0, "mass": st.mass.copy(), "vol0": st.vol0.copy()}
    out.update(state_arrays(st, "in"))
    for it in range(1, 101):
        sm.substep(st, mats, params)
        if it in (1, 10, 100):
            out.update(state_arrays(st, f"s{it}"))
    np.savez_compressed(os.path.join(OUT, "floor_block.npz"), **out)


def spec_reference():
    rng = np.random.default_rng(11)
    grid = sm.Grid(resolution=(16, 16, 16))
    mats = [sm.Material(5e3, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.3, 0.5), (0.25, 0.25, 0.25), 512, seed=42, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    st.C[:] = rng.normal(0, 1.0, st.C.shape)
    st.F[:] = np.eye(3) + rng.normal(0, 0.05, st.F.shape)
    mu, lam, _ = sm.materials.pack_materials(mats)
    out = {"res": np.array(grid.resolution), "extent": np.array(grid.extent),
           "E": 5e3, "nu": 0.3, "rho": 1000.0, "mass": st.mass.copy(), "vol0": st.vol0.copy()}
    out.update(state_arrays(st, "in"))
    _, hi = grid.margin_bounds()
    for _ in range(5):
        reference_substep(st.x, st.v, st.F, st.C, st.mass, st.vol0, st.material_id, mu, lam,
                          st.grid_mv, st.grid_m, 5e-4, grid.dx, 0.0, -9.8, 0.0, 3, False,
                          hi[0], hi[1], hi[2])
    out.update(state_arrays(st, "s5"))
    np.savez_compressed(os.path.join(OUT, "spec_reference.npz"), **out)


def stage_ops():
    rng = np.random.default_rng(1234)
    grid = sm.Grid(resolution=(16, 16, 16))
    n = 300
    lo, hi = grid.margin_bounds()
    st = sm.SimState(grid=grid, x=rng.uniform(lo + 0.02, hi - 0.02, (n, 3)),
                     v=rng.normal(0, 0.5, (n, 3)),
                     F=np.tile(np.eye(3), (n, 1, 1)) + rng.normal(0, 0.05, (n, 3, 3)),
                     C=rng.normal(0, 2.0, (n, 3, 3)), mass=rng.uniform(1e-4, 2e-3, n),
                     vol0=rng.uniform(1e-7, 1e-6, n), material_id=np.zeros(n, np.int32))
    mats = [sm.Material(5e3, 0.3, 1000.0)]
    params = sm.SimParams()
    out = {"res": np.array(grid.resolution), "extent": np.array(grid.extent),
           "E": 5e3, "nu": 0.3, "rho": 1000.0, "mass": st.mass.copy(), "vol0": st.vol0.copy()}
    out.update(state_arrays(st, "in"))
    out["p2g_inverted"] = sm.p2g(st, mats, params)
    out["p2g_F"] = st.F.copy()
    out["p2g_grid_mv"] = st.grid_mv.copy()
    out["p2g_grid_m"] = st.grid_m.copy()
    sm.grid_update(st, params)
    out["gu_grid_mv"] = st.grid_mv.copy()
    sm.g2p_advect(st, params)
    out.update(state_arrays(st, "g2p"))
    np.savez_compressed(os.path.join(OUT, "stage_ops.npz"), **out)


def kinematics():
    q0 = Rotation.from_euler("xyz", [10, 20, 30], degrees=True).as_quat()
    q1 = Rotation.from_euler("xyz", [40, -10, 75], degrees=True).as_quat()
    q2 = Rotation.from_euler("y", 90, degrees=True).as_quat()
    traj = [sm.Keyframe(0.0, [(np.array([0.5, 0.45, 0.5]), q0)]),
            sm.Keyframe(0.3, [(np.array([0.5, 0.2, 0.4]), q1)], jaw_state="closed"),
            sm.Keyframe(0.7, [(np.array([0.6, 0.3, 0.5]), q2)])]
    times = np.array([-0.1, 0.0, 0.0125, 0.1, 0.2999, 0.3, 0.45, 0.6999, 0.7, 1.0])
    T, R, lv, av, jaw = [], [], [], [], []
    for t in times:
        poses, j = sm.pose_at(traj, float(t))
        T.append(poses[0][0]); R.append(poses[0][1]); lv.append(poses[0][2]); av.append(poses[0][3])
        jaw.append(1 if j == "closed" else 0)
    spawn = sm.sample_box((0.5, 0.2, 0.5), (0.3, 0.1, 0.2), 1000, seed=5)
    np.savez_compressed(os.path.join(OUT, "kinematics.npz"), times=times,
                        key_t=np.array([0.0, 0.3, 0.7]), key_T=np.array([[0.5, 0.45, 0.5],
                                                                          [0.5, 0.2, 0.4],
                                                                          [0.6, 0.3, 0.5]]),
                        key_q=np.array([q0, q1, q2]), key_jaw=np.array([0, 1, 0]),
                        T=np.array(T), R=np.array(R), lv=np.array(lv), av=np.array(av),
                        jaw=np.array(jaw), sample_positions=spawn.positions,
                        sample_volume=spawn.rest_volume_per_particle)


def frame_ops():
    grid = sm.Grid(resolution=(16, 16, 16), extent=(1.0, 1.0, 1.0))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.5, 0.5), (0.3, 0.3, 0.3), 4000, seed=21, grid=grid)
    blob = sm.SimState.from_spawns(grid, [spawn], mats)
    f16 = sm.splat_density(blob.x, blob.mass, grid)
    f32 = sm.splat_density(blob.x, blob.mass, grid, resolution=(32, 32, 32))
    g2 = sm.Grid(resolution=(32, 32, 32), extent=(1.0, 1.0, 1.0))
    st = sm.SimState.from_spawns(g2, [sm.sample_box((0.5, 0.14, 0.5), (0.3, 0.16, 0.3), 3000, seed=4,
                                                    grid=g2)], mats)
    x0 = st.x.copy()
    params = sm.SimParams()
    for _ in range(40):
        sm.substep(st, mats, params)
    st.x[:200, 1] += 3.0 * g2.dx  # some lifted / detached particles
    m = sm.compute_metrics(st, x0)
    np.savez_compressed(os.path.join(OUT, "frame_ops.npz"), blob_x=blob.x, blob_mass=blob.mass,
                        splat16=f16.values, splat16_dx=f16.dx, splat32=f32.values, splat32_dx=f32.dx,
                        met_x0=x0, met_x=st.x, met_F=st.F, met_dx=g2.dx,
                        met=np.array([m.lifted_fraction, m.detached_fraction, m.mean_abs_j_minus_1,
                                      m.max_displacement]))


def mpmf_frame():
    """server.encode_frame bytes for a small mesh (with and without normals /
    UVs) and two collider records, plus the inputs."""
    from softmpm import server
    rng = np.random.default_rng(11)
    v = rng.uniform(-1.0, 2.0, (37, 3))
    n = rng.normal(size=(37, 3))
    uv = rng.uniform(0.0, 1.0, (37, 2))
    t = rng.integers(0, 37, (50, 3)).astype(np.int32)
    cols = [server.ColliderPose(0, np.array([0.1, 0.2, 0.3]), np.array([0.0, 0.0, 0.0, 1.0]), False),
            server.ColliderPose(5, np.array([-1.5, 2.25, 1e-3]), np.array([0.1, -0.2, 0.3, 0.927]), True)]
    full = server.encode_frame(sm.SurfaceMesh(vertices=v, indices=t, uvs=uv, normals=n), cols, 42, 1.0 / 3.0)
    bare = server.encode_frame(sm.SurfaceMesh(vertices=v, indices=t), [], 7, 0.5)
    np.savez_compressed(os.path.join(OUT, "mpmf_frame.npz"), v=v, n=n, uv=uv, t=t,
                        col_id=np.array([c.id for c in cols]), col_t=np.array([c.translation for c in cols]),
                        col_q=np.array([c.quaternion for c in cols]), col_jaw=np.array([c.jaw_closed for c in cols]),
                        full=np.frombuffer(full, np.uint8), bare=np.frombuffer(bare, np.uint8))


if __name__ == "__main__":
    mpmf_frame()
    frame_ops()
    substep_colliders()
    floor_block()
    spec_reference()
    stage_ops()
    kinematics()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
