# quick GPU check: parity subset + C3 bench line (no CPU baseline)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenes.py -x -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('C3', round(d['value']/1e9,3), 'ms/frame', round(d['ms_per_step'],3), 'fused', round(k['fused_mean']*1e3,1), 'grid', round(k['grid_op_mean']*1e3,2), 'frac', round(d['roofline']['frac'],3), 'sm', d['clocks']['sm_mhz'])"
