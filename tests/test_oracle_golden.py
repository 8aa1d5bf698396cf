"""The CPU oracle (oracle/mpm_oracle.c) against golden vectors produced by the
REAL reference package (tests/golden/make_golden.py).  O1 must be bit-exact:
same arithmetic order as the numba kernels, fastmath off."""
import numpy as np

from conftest import load_golden, packed_from_golden
from oracle import oracle as O
from paper_2402_01181_b200.materials import Material


def _sim(g, chunks=8, theta=-1.0, stress_form=0):
    res = tuple(int(r) for r in g["res"])
    dx = float(g["extent"][0]) / res[0]
    m = Material(float(g["E"]), float(g["nu"]), float(g["rho"]))
    p = O.OracleParams(res=res, dx=dx, theta=theta, chunks=chunks, stress_form=stress_form)
    return O.OracleSim(p, g["in_x"], g["in_v"], g["in_F"], g["in_C"], g["mass"], g["vol0"],
                       np.zeros(len(g["in_x"]), np.int32), m.mu, m.lam)


def test_o1_substep_with_colliders_bit_exact():
    g = load_golden("substep_colliders.npz")
    res = tuple(int(r) for r in g["res"])
    dx = float(g["extent"][0]) / res[0]
    sim = _sim(g, theta=0.5 * dx)
    packed = packed_from_golden(g)
    inv = sim.substep(packed)
    assert inv == int(g["s1_inverted"])
    for k in ("x", "v", "F", "C"):
        assert np.array_equal(getattr(sim, k), g[f"s1_{k}"]), k
    assert np.array_equal(sim.grid_mv, g["s1_grid_mv"])
    assert np.array_equal(sim.grid_m, g["s1_grid_m"])
    dist, obj = sim.collision_field(packed, 0.5 * dx)
    assert np.array_equal(dist, g["s1_dist"])
    assert np.array_equal(obj, g["s1_obj"])
    for _ in range(9):
        sim.substep(packed)
    for k in ("x", "v", "F", "C"):
        assert np.array_equal(getattr(sim, k), g[f"s10_{k}"]), k


def test_o1_floor_block_trajectory_bit_exact():
    g = load_golden("floor_block.npz")
    sim = _sim(g)
    for it in range(1, 101):
        sim.substep(None)
        if it in (1, 10, 100):
            for k in ("x", "v", "F", "C"):
                assert np.array_equal(getattr(sim, k), g[f"s{it}_{k}"]), (it, k)


def test_o1_result_independent_of_thread_count():
    g = load_golden("floor_block.npz")
    outs = []
    before = O.max_threads()
    try:
        for t in (1, 3):
            O.set_threads(t)
            sim = _sim(g)
            for _ in range(5):
                sim.substep(None)
            outs.append(sim.x.copy())
    finally:
        O.set_threads(before)
    assert np.array_equal(outs[0], outs[1])


def test_o2_spec_reference_bit_exact():
    g = load_golden("spec_reference.npz")
    res = tuple(int(r) for r in g["res"])
    dx = float(g["extent"][0]) / res[0]
    m = Material(float(g["E"]), float(g["nu"]), float(g["rho"]))
    x, v, F, C = (np.array(g[f"in_{k}"]) for k in "xvFC")
    gmv = np.zeros(res + (3,))
    gm = np.zeros(res)
    hi = tuple((r - 1.5 - 1e-7) * dx for r in res)
    for _ in range(5):
        O.reference_substep(x, v, F, C, g["mass"], g["vol0"], np.zeros(len(x), np.int32), m.mu,
                            m.lam, gmv, gm, 5e-4, dx, (0.0, -9.8, 0.0), 3, False, hi)
    for k, a in zip("xvFC", (x, v, F, C)):
        assert np.array_equal(a, g[f"s5_{k}"]), k


def test_o3_fp32_sorted_close_to_o1_and_conserves_mass():
    g = load_golden("stage_ops.npz")
    res = tuple(int(r) for r in g["res"])
    dx = float(g["extent"][0]) / res[0]
    m = Material(float(g["E"]), float(g["nu"]), float(g["rho"]))
    order = O.sorted_order(np.float32(g["in_x"]), dx, res)
    gmv, gm, F, inv = O.p2g_sorted_fp32(g["in_x"], g["in_v"], g["in_F"], g["in_C"], g["mass"],
                                         g["vol0"], np.zeros(len(order), np.int32), m.mu, m.lam,
                                         5e-4, dx, res, order)
    assert inv == int(g["p2g_inverted"])
    assert abs(gm.astype(np.float64).sum() - g["mass"].sum()) / g["mass"].sum() < 1e-6
    assert np.abs(gm - g["p2g_grid_m"]).max() <= 1e-6 * np.abs(g["p2g_grid_m"]).max()
    scale = np.abs(g["p2g_grid_mv"]).max()
    assert np.abs(gmv - g["p2g_grid_mv"]).max() <= 1e-5 * scale
    assert np.abs(F - g["p2g_F"]).max() < 1e-6
    # order matters for fp32 sums: a different order gives different bits somewhere
    _, gm2, _, _ = O.p2g_sorted_fp32(g["in_x"], g["in_v"], g["in_F"], g["in_C"], g["mass"],
                                     g["vol0"], np.zeros(len(order), np.int32), m.mu, m.lam,
                                     5e-4, dx, res, order[::-1].copy())
    assert np.abs(gm2 - gm).max() <= 1e-6 * gm.max()


def test_oracle_splat_density_bit_exact():
    """surfacing.splat_density (kernels.py:541-588) on the test_surfacing blob,
    on the sim lattice and a 2x finer one."""
    g = load_golden("frame_ops.npz")
    for key, res in (("splat16", (16, 16, 16)), ("splat32", (32, 32, 32))):
        out = O.splat_density(g["blob_x"], g["blob_mass"], res, float(g[f"{key}_dx"]))
        assert np.array_equal(out, g[key]), key
    assert np.abs(O.splat_density(np.zeros((0, 3)), np.zeros(0), (16, 16, 16), 1 / 16)).max() == 0.0


def test_oracle_compute_metrics_exact():
    g = load_golden("frame_ops.npz")
    got = O.compute_metrics(g["met_x"], g["met_F"], g["met_x0"], float(g["met_dx"]))
    assert np.array_equal(np.array(got), g["met"])
