"""Bitwise self-check of the exact-arithmetic shortcuts in collide.cuh (the
square root and divisions skipped at box faces) against the reference's plain
formulas (kernels.py:30-45, 116-158) on 16 M points near faces, edges and
corners of rotated boxes; the harness is compiled with nvcc on the box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_box_distance_and_normal_shortcuts_are_bit_exact(tmp_path):
    exe = tmp_path / "collide_exact"
    subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                    os.path.join(HERE, "cuda", "collide_exact.cu")], check=True, capture_output=True, timeout=300)
    out = subprocess.run([str(exe), str(1 << 24)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    fields = out.stdout.split()
    assert int(fields[3]) == 0 and int(fields[5]) > (1 << 22), out.stdout   # mismatches, fast-path hits
