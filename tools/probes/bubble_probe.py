"""Inter-kernel bubbles of the C3 frame without per-kernel events (run with
SOFTMPM_LIB pointing at the profile build: `make -C paper_2402_01181_b200/csrc
profile`; the counters print when the context is destroyed)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2402_01181_b200 as sm  # noqa: E402

st, mats, params, cols, pose_fn = bench.build_scene("c3", None, 1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    sm.step(st, mats, params, cols, pose_fn)
del st  # Context.__del__ -> mpm_destroy prints the profile counters
import gc
gc.collect()
