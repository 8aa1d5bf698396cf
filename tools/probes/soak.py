"""Long-horizon soak of a bench scene: N frames through the public API, then
NaN / mass / bounds / inverted-element checks (robustness, not a measurement).
    python tools/probes/soak.py c3 200"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2402_01181_b200 as sm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 200
st, mats, params, cols, pose_fn = bench.build_scene(cfg, None, 1)
m0 = float(st.mass.sum())
t0 = time.perf_counter()
inv = 0
for f in range(frames):
    rep = sm.step(st, mats, params, cols, pose_fn)
    inv += rep.inverted_particles
    if (f + 1) % 50 == 0:
        nan = st.has_nan()
        x = st.x
        lo, hi = st.grid.margin_bounds()
        print(f"frame {f + 1}: t={st.time:.4f} nan={nan} x in [{x.min():.4f}, {x.max():.4f}] "
              f"(margin [{np.min(lo):.4f}, {np.max(hi):.4f}]) inverted so far {inv} "
              f"mean|J-1|={np.abs(np.linalg.det(st.F) - 1).mean():.3e}", flush=True)
        assert not nan
print(f"{frames} frames in {time.perf_counter() - t0:.1f} s; mass drift {abs(float(st.mass.sum()) - m0) / m0:.2e}")
