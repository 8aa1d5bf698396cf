# A/B of library builds on one box: bash tools/sweeps/ab.sh NAME=path.so ... (env passes through)
# Alternates the builds ROUNDS times (default 3) and prints each run; compare medians.
ROUNDS=${ROUNDS:-3}
STEPS=${STEPS:-20}
CONFIG=${CONFIG:-c3}
for r in $(seq $ROUNDS); do
  for kv in "$@"; do
    name=${kv%%=*}; lib=${kv#*=}
    SOFTMPM_LIB=$lib python bench.py --config $CONFIG --steps $STEPS --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('$name', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'fused', round(k['fused_mean']*1e3,1), 'grid', round(k['grid_op_mean']*1e3,2), 'items', k['work_items'], 'sm', d['clocks']['sm_mhz'])"
  done
done
