"""The reference package's OWN hot-path tests, run through install().

tools/install_reference.sh installs the unmodified reference (softmpm) into
baseline/_ref and copies its tests/test_transfers.py, test_substep.py,
test_collision.py, test_weights.py, test_materials.py and test_oracle.py
(/root/reference/pkg/tests) beside it.  tools/ref_suite/ref_suite_plugin.py
imports that softmpm, calls paper_2402_01181_b200.install(softmpm) -- so
softmpm.p2g / grid_update / g2p_advect / substep / step run on the B200
kernels -- and maps the tests' fp64 tolerance literals (< 1e-5 on the right
of a < / <= comparison or as an approx / allclose tolerance) to the fp32
gate 1e-5.  The test runs that suite in a subprocess, in the fast mode and
in the deterministic mode, and requires every test to pass except the ones
listed in MAY_FAIL for that mode, with the reason.""" 
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
MODULES = ["test_transfers.py", "test_substep.py", "test_collision.py", "test_weights.py",
           "test_materials.py", "test_oracle.py",
           # the callers and data formats either side of the path: surfacing,
           # scene build + metrics, the CLI, the acceptance suite, sampling, SDF, the server
           "test_surfacing.py", "test_scene.py", "test_cli.py", "test_acceptance.py", "test_sampling.py",
           "test_sdf.py", "test_server.py"]
# tests allowed to fail per install mode, with the reason (documented in DESIGN.md)
_ORDER = ("fast mode flushes its fixed-point tiles into the grid with float L2 reductions in "
          "arrival order, so runs agree to fp32 rounding, not bit for bit (SURVEY 8d: not required "
          "in fast mode); install(deterministic=True) is bitwise reproducible")
_NOT_OURS = {
    "test_server.py::test_golden_fixture_matches_current_encoder":
        "the reference package ships frontend/test/fixtures/golden_frame.bin's generator outside pkg/src "
        "(fails on the reference itself, SURVEY 4)",
    "test_acceptance.py::test_sdf_fidelity_256":
        "wall-clock budget of the reference's CPU numba SDF bake (off the hot path; 11.4 s vs 10 s on the "
        "reference itself, SURVEY 4)",
    "test_cli.py::test_multithread_not_slower_at_scale":
        "times the reference's numba thread-count knob, which the GPU path does not use",
    "test_acceptance.py::test_scaling_trend_single_thread":
        "fits the reference's single-thread CPU ms/frame against particle count (R^2); through install() "
        "a 6-48 K particle frame takes 1-2 ms, dominated by fixed launch / transfer costs, so the fit is "
        "noise (it passes or fails from run to run)",
}
MAY_FAIL = {
    "fast": {"test_substep.py::test_runs_are_bitwise_deterministic": _ORDER,
             "test_substep.py::test_determinism_across_thread_counts": _ORDER,
             "test_server.py::test_session_pause_resume_reset": _ORDER + " (compares two sessions bit for bit)",
             "test_cli.py::test_run_is_reproducible": _ORDER + " (compares two CLI runs' metrics.csv bytes)",
             **_NOT_OURS},
    "deterministic": dict(_NOT_OURS),
}


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "ref_tests")),
                    reason="reference not installed (bash tools/install_reference.sh)")
@pytest.mark.parametrize("mode", ["fast", "deterministic"])
def test_reference_hot_path_suite_through_install(mode):
    env = dict(os.environ)
    env["SOFTMPM_INSTALL_DETERMINISTIC"] = "1" if mode == "deterministic" else "0"
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tools", "ref_suite"), REF, ROOT,
                                         env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")
    files = [os.path.join(REF, "ref_tests", m) for m in MODULES]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-rA", "-p", "ref_suite_plugin",
                        "-p", "no:cacheprovider", "--rootdir", os.path.join(REF, "ref_tests"), *files],
                       cwd=os.path.join(REF, "ref_tests"), env=env, capture_output=True, text=True,
                       timeout=2400)
    out = r.stdout + r.stderr
    print(out[-8000:])
    assert "install() active: True" in out and f"install mode: {mode}" in out
    failed = [ln.split()[1] for ln in out.splitlines() if ln.startswith(("FAILED ", "ERROR "))]
    failed = [os.path.basename(f) for f in failed]
    unexpected = [f for f in failed if f not in MAY_FAIL[mode]]
    assert not unexpected, unexpected
    passed = sum(1 for ln in out.splitlines() if ln.startswith("PASSED "))
    assert passed >= 125, passed


def _import_reference():
    import types
    if "skimage" not in sys.modules:
        sk = types.ModuleType("skimage")
        sk.measure = types.ModuleType("skimage.measure")
        sys.modules["skimage"], sys.modules["skimage.measure"] = sk, sk.measure
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")
    if REF not in sys.path:
        sys.path.append(REF)
    import softmpm
    return softmpm


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "softmpm")),
                    reason="reference not installed (bash tools/install_reference.sh)")
def test_install_writes_back_collision_field_and_grid_lazily():
    """install() on the real reference: after softmpm.step with a tool,
    state._collision is the merged field of the last substep (core.py:307-309,
    read by demos/02_tool_contact.py:39) and the dense grid arrives on first
    read; uninstall() restores the class."""
    import numpy as np
    import paper_2402_01181_b200 as b200
    ref = _import_reference()
    had = "_collision" in ref.core.SimState.__dict__
    b200.install(ref)
    try:
        grid = ref.Grid(resolution=(32, 32, 32), extent=(1.0, 1.0, 1.0))
        mats = [ref.Material(1.0e4, 0.3, 1000.0)]
        spawn = ref.sample_box((0.5, 0.14, 0.5), (0.3, 0.16, 0.3), 4000, seed=1, grid=grid)
        st = ref.SimState.from_spawns(grid, [spawn], mats)
        tool = ref.RigidCollider(id=0, shape=ref.Box(np.array([0.08, 0.03, 0.08])),
                                 translation=np.array([0.5, 0.235, 0.5]),
                                 linear_velocity=np.array([0.0, -0.5, 0.0]), friction_mu=0.4)
        rep = ref.step(st, mats, ref.SimParams(), [tool])
        assert rep.step_index == 1
        assert "grid_mv" in st.__dict__.get("_b200_stale", set())   # not copied yet
        col = st._collision
        assert col is not None and (col.object_id >= 0).sum() > 0
        assert col.distance.shape == grid.resolution
        assert abs(st.grid_m.sum() - st.mass.sum()) < 1e-5 * st.mass.sum()
        assert "grid_m" not in st.__dict__["_b200_stale"]
    finally:
        b200.uninstall(ref)
    assert ("_collision" in ref.core.SimState.__dict__) == had
