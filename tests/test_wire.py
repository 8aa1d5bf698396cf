"""MPMF frame codec (server.py:36-124) against the reference's own encoder:
golden bytes from tests/golden/make_golden.py (mpmf_frame)."""
import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from conftest import load_golden
from paper_2402_01181_b200 import wire
from paper_2402_01181_b200.errors import SimError


def _golden():
    g = load_golden("mpmf_frame.npz")
    cols = [wire.ColliderPose(int(i), t, q, bool(j)) for i, t, q, j in zip(g["col_id"], g["col_t"], g["col_q"],
                                                                            g["col_jaw"])]
    return g, cols


def test_encode_frame_matches_reference_bytes():
    g, cols = _golden()
    full = sm.encode_frame(sm.SurfaceMesh(vertices=g["v"], indices=g["t"], uvs=g["uv"], normals=g["n"]), cols, 42,
                           1.0 / 3.0)
    assert full == g["full"].tobytes()
    bare = sm.encode_frame(sm.SurfaceMesh(vertices=g["v"], indices=g["t"]), [], 7, 0.5)
    assert bare == g["bare"].tobytes()


def test_decode_is_the_inverse():
    g, cols = _golden()
    d = sm.decode_frame(g["full"].tobytes())
    assert d.frame_index == 42 and d.sim_time == np.float32(1.0 / 3.0)
    assert np.array_equal(d.vertices, g["v"].astype(np.float32)) and np.array_equal(d.indices, g["t"])
    assert np.array_equal(d.uvs, g["uv"].astype(np.float32)) and np.array_equal(d.normals, g["n"].astype(np.float32))
    assert [c.id for c in d.colliders] == [0, 5] and d.colliders[1].jaw_closed
    assert np.allclose(d.colliders[1].quaternion, g["col_q"][1], atol=1e-7)


def test_decode_rejects_bad_magic_and_trailing_bytes():
    g, _ = _golden()
    data = g["bare"].tobytes()
    with pytest.raises(SimError):
        sm.decode_frame(b"XXXX" + data[4:])
    with pytest.raises(SimError):
        sm.decode_frame(data + b"\0")


def test_frame_too_large(monkeypatch):
    monkeypatch.setattr(wire, "MAX_VERTICES", 4)
    mesh = sm.SurfaceMesh(vertices=np.zeros((5, 3)), indices=np.zeros((1, 3), np.int32))
    with pytest.raises(wire.FrameTooLarge):
        sm.encode_frame(mesh, [], 0, 0.0)
