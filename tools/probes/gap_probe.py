"""Per-frame device time: frame-by-frame (sync between frames, as bench.py)
vs back-to-back frames (host launch overhead hidden behind the GPU)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2402_01181_b200 import core as C  # noqa: E402

st, mats, params, cols, pose_fn = bench.build_scene("c3", None, 1)
for _ in range(3):
    C.step(st, mats, params, cols, pose_fn)
ctx = st._ctx
rows = bench.pose_rows(st, cols, params, pose_fn, st.time)
st._upload_pose_rows(*rows)


def frame():
    inv = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    ctx.call("mpm_substeps", 25, 1, ctypes.byref(inv), ctypes.byref(ms))
    return ms.value


frame()
torch.cuda.synchronize()
per = [frame() for _ in range(20)]
print("frame-by-frame (mpm events):", round(sum(per) / len(per), 4), "ms")
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
s.record(torch.cuda.current_stream())
for _ in range(20):
    inv = ctypes.c_int64(0)
    ctx.call("mpm_substeps", 25, 1, ctypes.byref(inv), None)
torch.cuda.synchronize()
print("back-to-back wall:", round((time.perf_counter() - t0) / 20 * 1e3, 4), "ms per frame")
