# grid-op launch shape A/B (run on the GPU box from the repo root)
L=$PWD/paper_2402_01181_b200
run() { python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('$1', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(k['fused_mean']*1e3,1), round(k['grid_op_mean']*1e3,2))"; }
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenes.py -q -x 2>&1 | tail -1
for g in 4 8; do SOFTMPM_GRIDOP_BLOCKS=$g run "minb4 blocks=$g"; done
for mb in 2 3; do for g in $mb 8; do SOFTMPM_LIB=$L/libsoftmpm_b200_g$mb.so SOFTMPM_GRIDOP_BLOCKS=$g run "minb$mb blocks=$g"; done; done
