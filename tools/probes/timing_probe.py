import ctypes, time, torch, sys
sys.path.insert(0, '.')
from paper_2402_01181_b200 import scenes
from paper_2402_01181_b200 import _lib
L = _lib.lib()
from paper_2402_01181_b200 import core
st, mats, params, cols, pose_fn = scenes.c3()
rep = core.step(st, mats, params, cols, pose_fn)
ctx = st._ctx
def frames(k, timing):
    L.mpm_set_timing(ctx.h, timing)
    tot = 0.0
    for _ in range(k):
        inv = ctypes.c_int64(0); ms = ctypes.c_double(0)
        ctx.call("mpm_substeps", 25, 1, ctypes.byref(inv), ctypes.byref(ms))
        tot += ms.value
    L.mpm_set_timing(ctx.h, 0)
    return tot / k
for t in (0, 1, 0, 1):
    frames(3, t)
    print("timing", t, "ms/frame", round(frames(20, t), 4))
