"""Full-size parity of the headline configurations against the CPU oracle O1
(fp64 restatement of the reference kernels, /root/reference/pkg/src/softmpm/
kernels.py:161-534 via core.step, core.py:280-320), fed the same per-substep
tool poses.

  * C3 (the bench workload): 1 M particles, 256^3, box tool pressing -- the
    exact scene bench.py times (scenes.c3 defaults);
  * C2: 30 K particles, 128^3, two baked-SDF capsule jaws (SDF 64^3) going
    down, closing (sticky) and pulling, in the reference's frozen-mode
    semantics and in live mode; 36 frames so the jaws close.

Gates (BASELINE north star): rel-L2 of x, v, F <= 1e-5 after the first
substep and <= 1e-3 after >= 100 substeps; C as |dC| dx / |v| <= 5e-5 after
the first substep."""
import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import scenes
from conftest import rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL_1 = 1e-5
TOL_100 = 1e-3
TOL_C = 5e-5


def _oracle_for(st, mats):
    g = st.grid
    O.set_threads(O.max_threads())
    return O.OracleSim(O.OracleParams(res=g.resolution, dx=g.dx, theta=0.5 * g.dx),
                       st.x, st.v, st.F, st.C, st.mass, st.vol0, st.material_id, mats[0].mu,
                       mats[0].lam)


class _Pair:
    """GPU state + oracle advanced frame by frame with identical poses."""

    def __init__(self, build, live=False, **kw):
        self.st, self.mats, _, self.cols, self.pose_fn = build(**kw)
        _, _, _, self.ocols, _ = build(**kw)
        self.osim = _oracle_for(self.st, self.mats)
        self.live = live
        self.packed = None
        self.t = 0.0

    def frames(self, n, substeps=25):
        params = sm.SimParams(substeps_per_frame=substeps,
                              collider_mode="live" if self.live else "frozen")
        for _ in range(n):
            sm.step(self.st, self.mats, params, self.cols, self.pose_fn)
            for _ in range(substeps):
                self.pose_fn(self.ocols, self.t)
                if self.packed is None or self.live:
                    self.packed = sm.pack_colliders(self.ocols)
                else:
                    self.packed.refresh_poses(self.ocols)  # reference: mode frozen at first pack
                self.osim.substep(self.packed)
                self.t += params.dt
        assert self.st.time == pytest.approx(self.t, rel=1e-12)

    def errors(self):
        e = {k: rel_l2(getattr(self.st, k), getattr(self.osim, k)) for k in ("x", "v", "F")}
        e["C"] = float(np.linalg.norm(self.st.C - self.osim.C) * self.st.grid.dx /
                       max(np.linalg.norm(self.osim.v), 1e-30))
        return e


def test_c3_full_size_matches_oracle():
    """The bench scene itself: 1 M particles on 256^3 with the pressing tool,
    first substep <= 1e-5, then 100 more substeps (4 frames) <= 1e-3."""
    pair = _Pair(scenes.c3)
    assert pair.st.particle_count == 1_000_000 and pair.st.grid.resolution == (256, 256, 256)
    pair.frames(1, substeps=1)
    e1 = pair.errors()
    print("c3 after 1 substep", e1)
    for k in ("x", "v", "F"):
        assert e1[k] < TOL_1, (k, e1)
    assert e1["C"] < TOL_C, e1
    pair.frames(4)
    e = pair.errors()
    print("c3 after 101 substeps", e)
    for k in ("x", "v", "F"):
        assert e[k] < TOL_100, (k, e)
    assert (pair.st._collision.object_id >= 0).sum() > 0  # the tool is in contact by now
    assert not pair.st.has_nan()


@pytest.mark.parametrize("live", [False, True])
def test_c2_full_size_grasper_matches_oracle(live):
    """Config 2 at full size: 30 K particles, 128^3, SDF-64 capsule jaws; 36
    frames (900 substeps): the jaws descend, close at t = 0.35 s and pull."""
    pair = _Pair(scenes.c2, live=live, count=30_000, res=128, sdf_res=64)
    pair.frames(1, substeps=1)
    e1 = pair.errors()
    for k in ("x", "v", "F"):
        assert e1[k] < TOL_1, (k, e1)
    pair.frames(36)
    e = pair.errors()
    print(f"c2 live={live} after 901 substeps", e)
    assert (pair.st._collision.object_id >= 0).sum() > 0
    for k in ("x", "v", "F"):
        assert e[k] < TOL_100, (k, e)
    if live:
        assert [c.mode for c in pair.cols] == ["sticky", "sticky"]
    assert not pair.st.has_nan()


def test_mixed_pose_fn_frames_reuse_no_stale_graph():
    """step(pose_fn) and step() alternating on one state: each frame's graph
    must use its own pose table (the graph key includes the pose
    row count), matching the oracle fed the same poses."""
    st, mats, _, cols, pose_fn = scenes.c3(count=20_000, res=48)
    _, _, _, ocols, _ = scenes.c3(count=20_000, res=48)
    osim = _oracle_for(st, mats)
    params = sm.SimParams()
    packed = None
    t = 0.0
    for frame in range(6):
        with_fn = frame % 2 == 0
        sm.step(st, mats, params, cols, pose_fn if with_fn else None)
        for _ in range(params.substeps_per_frame):
            if with_fn:
                pose_fn(ocols, t)
            if packed is None:
                packed = sm.pack_colliders(ocols)
            else:
                packed.refresh_poses(ocols)
            osim.substep(packed)
            t += params.dt
    for k in ("x", "v", "F"):
        assert rel_l2(getattr(st, k), getattr(osim, k)) < TOL_100, k
