"""The C-ABI library loads and exports every symbol include/*.h declares."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2402_01181_b200 import _lib


def _declared():
    names = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            text = open(os.path.join(inc, f)).read()
            names |= set(re.findall(r"\b(mpm_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [n for n in sorted(declared) if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == declared


def test_library_is_sm100a_and_not_a_stub():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for kernel in ("fused_kernel", "grid_op_kernel", "g2p_kernel", "det_gather_kernel"):
        assert kernel in sass
    assert "REDG.E.ADD.F32x4" in sass  # vector L2 reductions of the tile flush


def test_version_and_create_without_device():
    L = _lib.lib()
    assert b"sm_100a" in L.mpm_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = _lib.MpmConfig()
    cfg.res = (ctypes.c_int * 3)(16, 16, 16)
    cfg.dx = 1 / 16
    cfg.dt = 5e-4
    h = ctypes.c_void_p()
    assert L.mpm_create(ctypes.byref(h), ctypes.byref(cfg)) == _lib.MPM_ECUDA
    cfg.res = (ctypes.c_int * 3)(4, 16, 16)
    assert L.mpm_create(ctypes.byref(h), ctypes.byref(cfg)) == _lib.MPM_EINVAL
