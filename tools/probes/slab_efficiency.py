"""Slab-decomposition overhead on one GPU: the same scene stepped as one
domain and as W peer-memory windows of one process (slab.step_local_peer:
the IPC halo kernels + device-counter protocol, migration per stretch), both
device-synchronised wall clock per frame.  All windows share the one GPU, so
the ratio (windows time / single-domain time) is the decomposition's extra
work per particle, not a scaling figure."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import torch

import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import slab


def scene(n, res):
    grid = sm.Grid((res, res, res))
    spawn = sm.sample_box((0.5, 0.065, 0.5), (0.4, 0.1, 0.4), n, seed=1, grid=grid)
    st = sm.SimState.from_spawns(grid, [spawn], [sm.Material(1.0e4, 0.3, 1000.0)])
    return grid, st


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 16_000_000
    res = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    windows = [int(w) for w in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 4]
    frames = 4
    mats = [sm.Material(1.0e4, 0.3, 1000.0)]
    params = sm.SimParams(dt=1.0e-4, rebin_interval=5)
    grid, st = scene(n, res)
    args = (st.x.copy(), st.v.copy(), st.F.copy(), st.C.copy(), st.mass.copy(), st.vol0.copy(),
            st.material_id.copy())
    sm.step(st, mats, params)  # warm-up (context, graphs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(frames):
        sm.step(st, mats, params)
    torch.cuda.synchronize()
    single = (time.perf_counter() - t0) / frames
    del st
    print(f"{n} particles, {res}^3, dt 1e-4, rebin every 5: single domain {single * 1e3:.2f} ms/frame "
          f"({n * 25 / single:.3e} particle-substeps/s)", flush=True)
    for W in windows:
        wins = slab.split_state(grid, *args, ranks=W, ghost_bricks=2)
        ex = slab.PeerExchange(wins)
        slab.step_local_peer(wins, ex, mats, params)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(frames):
            slab.step_local_peer(wins, ex, mats, params)
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / frames
        print(f"  {W} peer windows on one GPU: {el * 1e3:.2f} ms/frame = {el / single:.3f} x single domain "
              f"(windows {[w.state.particle_count for w in wins]})", flush=True)
        del wins, ex


if __name__ == "__main__":
    main()
