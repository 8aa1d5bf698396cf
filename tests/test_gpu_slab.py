"""Config 5 slab decomposition, emulated on one GPU: the scene cut into x-slab
windows (separate device contexts, halo exchange by device copies, particle
migration) must reproduce the undecomposed run (and the CPU oracle)."""
import numpy as np
import pytest

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import slab
from conftest import rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _scene(n=24000, res=64, seed=3):
    grid = sm.Grid((res, res, res))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    # a wide slab that sits across every cut, with sideways motion so particles migrate
    spawn = sm.sample_box((0.5, 0.16, 0.5), (0.8, 0.2, 0.5), n, seed=seed, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    rng = np.random.default_rng(seed)
    v = np.zeros((n, 3))
    v[:, 0] = 0.6 * np.sin(4.0 * np.pi * st.x[:, 0])  # +-0.6 m/s shear along x
    v[:, 1] = rng.normal(0, 0.05, n)
    return grid, mats, st.x.copy(), v, st.F.copy(), st.C.copy(), st.mass.copy(), st.vol0.copy(), \
        st.material_id.copy()


@pytest.mark.parametrize("ranks", [2, 3])
def test_slab_windows_match_single_domain(ranks):
    grid, mats, x, v, F, C, m, vol, mat = _scene()
    params = sm.SimParams(rebin_interval=5)
    ref = sm.SimState(grid, x, v, F, C, m, vol, mat)
    wins = slab.split_state(grid, x, v, F, C, m, vol, mat, ranks=ranks, ghost_bricks=2)
    assert sum(w.state.particle_count for w in wins) == len(x)
    ex = slab.LocalExchange(wins)
    osim = O.OracleSim(O.OracleParams(res=grid.resolution, dx=grid.dx), x, v, F, C, m, vol, mat,
                       mats[0].mu, mats[0].lam)
    for _ in range(4):
        slab.step_local(wins, ex, mats, params)
        sm.step(ref, mats, params)
        for _ in range(params.substeps_per_frame):
            osim.substep(None)
    gx, gv, gF, gC = slab.gather(wins, len(x))
    assert not np.isnan(gx).any(), "a particle got lost in migration"
    counts = [int(w.download()[0].size) for w in wins]
    assert sum(counts) == len(x)
    for k, a in (("x", gx), ("v", gv), ("F", gF)):
        assert rel_l2(a, getattr(ref, k)) < 1e-4, k
        assert rel_l2(a, getattr(osim, k)) < 1e-3, k
    # particles actually crossed the cuts
    base = np.floor(gx[:, 0] / grid.dx - 0.5)
    base0 = np.floor(x[:, 0] / grid.dx - 0.5)
    cuts = [w.own for w in wins]
    owner = lambda b: np.searchsorted([c[1] for c in cuts], b, side="right")
    assert (owner(base) != owner(base0)).sum() > 0


def _narrow_scene(n=40000, res=64, seed=5):
    """A block that spans only x in [0.3, 0.7] of the domain (equal
    x-slabs would leave the outer windows empty), sheared so particles migrate."""
    grid = sm.Grid((res, res, res))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.16, 0.5), (0.4, 0.2, 0.5), n, seed=seed, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    v = np.zeros((n, 3))
    v[:, 0] = 0.5 * np.sin(8.0 * np.pi * st.x[:, 0])
    return grid, mats, st.x.copy(), v, st.F.copy(), st.C.copy(), st.mass.copy(), st.vol0.copy(), \
        st.material_id.copy()


@pytest.mark.parametrize("ranks", [2, 4])
def test_peer_windows_match_single_domain(ranks):
    """Windows of one process exchanging halos through peer memory (the IPC
    kernels and device-counter protocol, no host sync per substep) on a scene
    that does not span the domain: balanced cuts, every window populated,
    particles migrate, the gathered state matches the undecomposed run."""
    grid, mats, x, v, F, C, m, vol, mat = _narrow_scene()
    params = sm.SimParams(rebin_interval=5)
    ref = sm.SimState(grid, x, v, F, C, m, vol, mat)
    wins = slab.split_state(grid, x, v, F, C, m, vol, mat, ranks=ranks, ghost_bricks=2)
    sizes = [w.state.particle_count for w in wins]
    assert min(sizes) > 0 and max(sizes) < 2.0 * len(x) / ranks, sizes
    ex = slab.PeerExchange(wins)
    for _ in range(4):
        slab.step_local_peer(wins, ex, mats, params)
        sm.step(ref, mats, params)
    gx, gv, gF, gC = slab.gather(wins, len(x))
    assert not np.isnan(gx).any(), "a particle got lost in migration"
    assert sum(int(w.download()[0].size) for w in wins) == len(x)
    for k, a in (("x", gx), ("v", gv), ("F", gF)):
        assert rel_l2(a, getattr(ref, k)) < 1e-4, k
    base = np.floor(gx[:, 0] / grid.dx - 0.5)
    base0 = np.floor(x[:, 0] / grid.dx - 0.5)
    hi = [w.own[1] for w in wins]
    owner = lambda b: np.searchsorted(hi, b, side="right")
    assert (owner(base) != owner(base0)).sum() > 0


def test_peer_windows_4m_particles_match_single_domain():
    """4 M particles on 256^3 cut into 2 peer-memory windows, 3 frames with
    migration, against the undecomposed run."""
    grid = sm.Grid((256, 256, 256))
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    spawn = sm.sample_box((0.5, 0.12, 0.5), (0.6, 0.15, 0.6), 4_000_000, seed=7, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], mats)
    x = st.x.copy()
    v = np.zeros_like(x)
    v[:, 0] = 0.4 * np.sin(6.0 * np.pi * x[:, 0])
    args = (x, v, st.F.copy(), st.C.copy(), st.mass.copy(), st.vol0.copy(), st.material_id.copy())
    del st
    params = sm.SimParams(rebin_interval=5)
    ref = sm.SimState(grid, *args)
    wins = slab.split_state(grid, *args, ranks=2, ghost_bricks=2)
    ex = slab.PeerExchange(wins)
    for _ in range(3):
        slab.step_local_peer(wins, ex, mats, params)
        sm.step(ref, mats, params)
    gx, gv, gF, _ = slab.gather(wins, len(x))
    assert not np.isnan(gx).any()
    for k, a in (("x", gx), ("v", gv), ("F", gF)):
        assert rel_l2(a, getattr(ref, k)) < 1e-4, k
