"""Two peer windows, 2 frames, for an ncu launch list of the slab path."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import slab
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 16_000_000
grid = sm.Grid((512, 512, 512))
spawn = sm.sample_box((0.5, 0.065, 0.5), (0.4, 0.1, 0.4), n, seed=1, grid=grid)
st = sm.SimState.from_spawns(grid, [spawn], [sm.Material(1.0e4, 0.3, 1000.0)])
mats = [sm.Material(1.0e4, 0.3, 1000.0)]
params = sm.SimParams(dt=1.0e-4, rebin_interval=5)
wins = slab.split_state(grid, st.x, st.v, st.F, st.C, st.mass, st.vol0, st.material_id, ranks=2)
del st
ex = slab.PeerExchange(wins)
for _ in range(3):
    slab.step_local_peer(wins, ex, mats, params)
torch.cuda.synchronize()
print("ok")
