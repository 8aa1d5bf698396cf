"""Particle transfer probe: mpm_upload_fields / mpm_download_particles times
for pinned and pageable fp64 host buffers, device-converted (host_xfer 0) vs
host-converted fp32 wire (host_xfer 1), at C3's particle count."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2402_01181_b200 as pk  # noqa: E402
from paper_2402_01181_b200 import _lib, scenes  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
st, mats, params, cols, pose_fn = scenes.c3(count=count)
pk.step(st, mats, params, cols, pose_fn)
ctx = st._ctx
L = _lib.lib()
n = st.particle_count
sizes = {"x": 3, "v": 3, "F": 9, "C": 9}
pinned, ptrs = {}, []
for k, w in sizes.items():
    p = L.mpm_host_alloc(n * w * 8)
    ptrs.append(p)
    pinned[k] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n * w,))
pageable = {k: np.empty(n * w) for k, w in sizes.items()}
mb = n * 24 * 8 / 1e6
for label, host in (("pinned", pinned), ("pageable", pageable)):
    args = [_lib.ptr(host[k]) for k in sizes]
    for mode in (0, 1):
        ctx.call("mpm_set_option", b"host_xfer", mode)
        ctx.call("mpm_download_particles", ctypes.c_uint32(15), *args)
        ctx.call("mpm_upload_fields", ctypes.c_uint32(15), *args)
        td, tu = [], []
        for _ in range(5):
            t = time.perf_counter()
            ctx.call("mpm_download_particles", ctypes.c_uint32(15), *args)
            td.append(time.perf_counter() - t)
            t = time.perf_counter()
            ctx.call("mpm_upload_fields", ctypes.c_uint32(15), *args)
            tu.append(time.perf_counter() - t)
        print(f"n={n} {label:9s} host_xfer={mode}: download {1e3 * min(td):.2f} ms ({mb / min(td) / 1e3:.1f} GB/s fp64), "
              f"upload {1e3 * min(tu):.2f} ms ({mb / min(tu) / 1e3:.1f} GB/s fp64)", flush=True)
# host conversion alone (numpy, one thread) for scale
a = pageable["F"]
t = time.perf_counter()
b = a.astype(np.float32)
print(f"numpy narrow 1 thread: {a.nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s of fp64")
for p in ptrs:
    L.mpm_host_free(p)
