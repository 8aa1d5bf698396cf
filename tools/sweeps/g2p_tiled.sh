timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_scenes.py tests/test_gpu_fullsize.py 2>&1 | tail -1
cat > /tmp/bitcheck.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2402_01181_b200 as sm
from paper_2402_01181_b200 import scenes
st, mats, params, cols, pose_fn = scenes.c3(count=200000, res=128)
for _ in range(3): sm.step(st, mats, params, cols, pose_fn)
np.savez(sys.argv[1], x=st.x, v=st.v, C=st.C, F=st.F)
PY
SOFTMPM_G2P_TILED=0 python /tmp/bitcheck.py /tmp/a.npz; SOFTMPM_G2P_TILED=1 python /tmp/bitcheck.py /tmp/b.npz
python -c "
import numpy as np; a=np.load('/tmp/a.npz'); b=np.load('/tmp/b.npz')
print({k: (np.array_equal(a[k], b[k]), float(np.abs(a[k]-b[k]).max())) for k in a.files})"
for r in 1 2; do for v in 0 1; do
  SOFTMPM_G2P_TILED=$v timeout 300 python bench.py --config c3 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('tiled=$v', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'g2p_total', round(k['g2p_total'],3))"
done; done
