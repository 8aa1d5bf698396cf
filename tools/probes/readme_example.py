import sys
sys.path.insert(0, ".")
import paper_2402_01181_b200 as sm
grid = sm.Grid(resolution=(256, 256, 256))
mats = [sm.Material(1.0e4, 0.3, 1000.0)]
state = sm.SimState.from_spawns(grid, [sm.sample_box((0.5, 0.1, 0.5), (0.5, 0.1, 0.5), 1_000_000,
                                                     seed=1, grid=grid)], mats)
tool = sm.RigidCollider(id=0, shape=sm.Box([0.08, 0.03, 0.08]), friction_mu=0.4)
pose_fn = sm.make_pose_fn([sm.Keyframe(0.0, [([0.5, 0.20, 0.5], [0, 0, 0, 1])]),
                           sm.Keyframe(0.07, [([0.5, 0.17, 0.5], [0, 0, 0, 1])])])
x0 = state.x.copy()
report = sm.step(state, mats, sm.SimParams(), [tool], pose_fn)
x = state.x
m = sm.compute_metrics(state, x0)
mesh = sm.extract_surface(state, iso=300.0)
frame = sm.encode_surface_frame(state, 300.0, [], 0, 0.0)
print(report, m, len(mesh.vertices), len(mesh.indices), len(frame))
