"""Particle transfers through the C ABI (mpm_upload_fields /
mpm_download_particles): every route -- fp64 over PCIe with device conversion,
the host-converted fp32 wire (pageable buffers, large transfers), large
pinned transfers with x / v crossing as fp64 beside it -- must produce the
same bits: the fp32 round-to-nearest of the caller's fp64 values, in the
caller's particle order (the device order is permuted by re-binning), and
MPM_DOWNLOAD_KEEP_EQUAL must keep exactly the destination values whose fp32
rounding equals the device's (core.py's in-place download,
test_transfers.py:121 of the reference)."""
import ctypes

import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import _lib, scenes

pytestmark = pytest.mark.gpu

WIDTH = {"x": 3, "v": 3, "F": 9, "C": 9}


def _values(rng, n, w, lo, hi):
    a = rng.uniform(lo, hi, n * w)
    # ties and edge values of the fp64 -> fp32 rounding
    k = min(len(a), 64)
    f = rng.uniform(0.2, 0.8, k).astype(np.float32).astype(np.float64)
    ulp = np.spacing(f.astype(np.float32)).astype(np.float64)
    a[:k] = f + 0.5 * ulp                      # exact ties: round to even
    a[k:2 * k] = (f + 0.5 * ulp * (1 + 2.0 ** -30))[: len(a[k:2 * k])]
    a[2 * k] = -0.0
    a[2 * k + 1] = 1.0e-40                     # fp32 subnormal after rounding
    a[2 * k + 2] = -3.0e-39
    return a


class _Pinned:
    def __init__(self, n):
        L = _lib.lib()
        self.ptrs, self.arr = [], {}
        for k, w in WIDTH.items():
            p = L.mpm_host_alloc(n * w * 8)
            assert p
            self.ptrs.append(p)
            self.arr[k] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n * w,))

    def free(self):
        for p in self.ptrs:
            _lib.lib().mpm_host_free(p)


def _state(n):
    st, mats, params, cols, pose_fn = scenes.c3(count=n, res=64)
    sm.step(st, mats, params, cols, pose_fn)  # re-binned: device order != caller order
    return st


@pytest.mark.parametrize("n", [20_000, 120_000])  # below / above the host-path size threshold
@pytest.mark.parametrize("host_xfer", [0, 1])
@pytest.mark.parametrize("pinned_up,pinned_down", [(False, False), (True, True), (True, False), (False, True)])
def test_round_trip_bits(n, host_xfer, pinned_up, pinned_down):
    st = _state(n)
    ctx = st._ctx
    ctx.call("mpm_set_option", b"host_xfer", host_xfer)
    rng = np.random.default_rng(n + 7 * host_xfer)
    src = {k: _values(rng, n, w, 0.2, 0.8) for k, w in WIDTH.items()}
    pin = _Pinned(n) if (pinned_up or pinned_down) else None
    try:
        up = {}
        for k in WIDTH:
            if pinned_up:
                pin.arr[k][:] = src[k]
                up[k] = pin.arr[k]
            else:
                up[k] = src[k]
        ctx.call("mpm_upload_fields", ctypes.c_uint32(15), *[_lib.ptr(up[k]) for k in WIDTH])
        if pinned_down:
            for k in WIDTH:
                pin.arr[k][:] = np.nan
            down = pin.arr
        else:
            down = {k: np.full(n * w, np.nan) for k, w in WIDTH.items()}
        ctx.call("mpm_download_particles", ctypes.c_uint32(15), *[_lib.ptr(down[k]) for k in WIDTH])
        for k in WIDTH:
            want = src[k].astype(np.float32).astype(np.float64)
            assert np.array_equal(down[k].view(np.uint64), want.view(np.uint64)), k
    finally:
        if pin:
            pin.free()


@pytest.mark.parametrize("n", [20_000, 120_000])
def test_keep_equal_download(n):
    st = _state(n)
    ctx = st._ctx
    rng = np.random.default_rng(3)
    src = {k: _values(rng, n, w, 0.2, 0.8) for k, w in WIDTH.items()}
    ctx.call("mpm_upload_fields", ctypes.c_uint32(15), *[_lib.ptr(src[k]) for k in WIDTH])
    # destination: the uploaded fp64 values, half of them perturbed beyond fp32 resolution
    dst = {k: v.copy() for k, v in src.items()}
    for k in WIDTH:
        dst[k][::2] += 1.0e-3
    keep = _lib.DOWNLOAD_KEEP_EQUAL
    ctx.call("mpm_download_particles", ctypes.c_uint32(15 | keep), *[_lib.ptr(dst[k]) for k in WIDTH])
    for k in WIDTH:
        dev = src[k].astype(np.float32)
        want = src[k].copy()                    # unperturbed: fp32(orig) == device -> orig kept
        want[::2] = dev[::2].astype(np.float64)  # perturbed: the device value
        assert np.array_equal(dst[k].view(np.uint64), want.view(np.uint64)), k
