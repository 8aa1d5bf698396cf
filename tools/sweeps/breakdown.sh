# per-kernel breakdown of several library builds (run on the GPU box from the repo root):
#   bash tools/sweeps/breakdown.sh NAME=path.so ...
for kv in "$@"; do
  name=${kv%%=*}; lib=${kv#*=}
  SOFTMPM_LIB=$lib python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; f=k['frames']
print('$name', 'value %.3e' % d['value'], 'ms/frame %.3f' % d['ms_per_step'], 'prof ms/frame %.3f' % (k['device_total']/f),
      'fused %.1f us x %.0f' % (k['fused_mean']*1e3, k['fused_launches']/f), 'A %.1f' % (k['g2p_stress_mean']*1e3),
      'B %.1f' % (k['p2g_tile_mean']*1e3), 'grid %.1f' % (k['grid_op_mean']*1e3), 'rebin/frame %.1f us' % (k['rebin_total']/f*1e3),
      'g2p/frame %.1f us' % (k['g2p_total']/f*1e3))"
done
