# work-item granularity sweep (run on the GPU box from the repo root)
run() { python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('$1', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'fused', round(k['fused_mean']*1e3,1), 'A', round(k['g2p_stress_mean']*1e3,1), 'B', round(k['p2g_tile_mean']*1e3,1), 'grid', round(k['grid_op_mean']*1e3,2), 'items', k['work_items'])"; }
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenes.py -q -x 2>&1 | tail -1
for i in ${ITEMS:-2 3 4 6 8}; do SOFTMPM_ITEMS_PER_SM=$i run "I=$i"; done
