"""Error growth of the GPU path vs O1 on colliding blocks (per frame)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np
import paper_2402_01181_b200 as sm
from oracle import oracle as O
from test_gpu_guard import _converging_blocks
from conftest import rel_l2

for speed in [float(a) for a in sys.argv[1:]] or [0.5, 1.5]:
    for split in (0, 1):
        st, mats = _converging_blocks(speed=speed)
        params = sm.SimParams(dt=2.0e-4, gravity=(0.0, 0.0, 0.0))
        g = st.grid
        O.set_threads(O.max_threads())
        osim = O.OracleSim(O.OracleParams(res=g.resolution, dx=g.dx, dt=2.0e-4, gravity=(0.0, 0.0, 0.0)), st.x, st.v, st.F, st.C,
                           st.mass, st.vol0, st.material_id, mats[0].mu, mats[0].lam)
        row = []
        for f in range(6):
            sm.step(st, mats, params)
            if f == 0 and split:
                st._ctx.call("mpm_set_option", b"split", 1)
            for _ in range(params.substeps_per_frame):
                osim.substep(None)
            e = [rel_l2(getattr(st, k), getattr(osim, k)) for k in ("x", "v", "F")]
            row.append(f"f{f}: x {e[0]:.1e} v {e[1]:.1e} F {e[2]:.1e} J {np.linalg.det(osim.F).min():.2f}")
        print(f"speed {speed} split {split}:", " | ".join(row), flush=True)
