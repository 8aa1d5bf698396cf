"""Diagnostic: frame-by-frame health of the C3 press scene (fast / deterministic / oracle)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import scenes
from oracle import oracle as O

count = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
res = int(sys.argv[2]) if len(sys.argv) > 2 else 64
frames = int(sys.argv[3]) if len(sys.argv) > 3 else 18
modes = sys.argv[4].split(",") if len(sys.argv) > 4 else ["fast", "det", "oracle"]
for mode in [m for m in modes if m != "oracle"]:
    st, mats, params, cols, pose_fn = scenes.c3(count=count, res=res)
    params = sm.SimParams(deterministic=(mode == "det"))
    for f in range(frames):
        rep = sm.step(st, mats, params, cols, pose_fn)
        x = st.x; F = st.F
        J = np.linalg.det(F)
        bad = st.has_nan()
        print(f"{mode} frame {f:2d} t={st.time:.4f} nan={bad} minJ={np.nanmin(J):.4f} maxv={np.nanmax(np.abs(st.v)):.3f} inv={rep.inverted_particles} toolY={cols[0].translation[1]:.4f}", flush=True)
        if bad:
            break
if 'oracle' not in modes:
    sys.exit(0)
st, mats, params, cols, pose_fn = scenes.c3(count=count, res=res)
g = st.grid
osim = O.OracleSim(O.OracleParams(res=g.resolution, dx=g.dx, theta=0.5 * g.dx), st.x, st.v, st.F, st.C,
                   st.mass, st.vol0, st.material_id, mats[0].mu, mats[0].lam)
t = 0.0
for f in range(frames):
    inv = 0
    for s in range(25):
        pose_fn(cols, t)
        inv += osim.substep(sm.pack_colliders(cols))
        t += params.dt
    J = np.linalg.det(osim.F)
    print(f"oracle frame {f:2d} nan={np.isnan(osim.x).any()} minJ={np.nanmin(J):.4f} maxv={np.nanmax(np.abs(osim.v)):.3f} inv={inv}", flush=True)
    if np.isnan(osim.x).any():
        break
