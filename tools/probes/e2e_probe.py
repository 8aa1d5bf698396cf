"""Where the e2e step time goes (C3, host fp64 buffers through the C ABI)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2402_01181_b200 import _lib  # noqa: E402
from paper_2402_01181_b200 import core as C  # noqa: E402

st, mats, params, cols, pose_fn = bench.build_scene("c3", None, 1)
C.step(st, mats, params, cols, pose_fn)
ctx = st._ctx
L = _lib.lib()
n = st.particle_count
sizes = {"x": 3, "v": 3, "F": 9, "C": 9}
host = {}
for k, w in sizes.items():
    p = L.mpm_host_alloc(n * w * 8)
    host[k] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n * w,))
ptrs = [_lib.ptr(host[k]) for k in sizes]
ctx.call("mpm_download_particles", ctypes.c_uint32(15), *ptrs)
acc = {"poses": 0.0, "upload": 0.0, "frame": 0.0, "download": 0.0}
K = 8
for it in range(K + 2):
    t0 = time.perf_counter()
    rows = bench.pose_rows(st, cols, params, pose_fn, st.time)
    st._upload_pose_rows(*rows)
    t1 = time.perf_counter()
    ctx.call("mpm_upload_fields", ctypes.c_uint32(15), *ptrs)
    t2 = time.perf_counter()
    inv = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    ctx.call("mpm_substeps", 25, 1, ctypes.byref(inv), ctypes.byref(ms))
    st.time += 25 * params.dt
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ctx.call("mpm_download_particles", ctypes.c_uint32(15), *ptrs)
    t4 = time.perf_counter()
    if it >= 2:
        for k, v in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            acc[k] += v / K
print({k: round(v * 1e3, 3) for k, v in acc.items()}, "total ms", round(sum(acc.values()) * 1e3, 3))
