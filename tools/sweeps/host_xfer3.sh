for r in 1 2 3; do
  for cfg in "0 0" "1 0" "1 1"; do
    set -- $cfg
    SOFTMPM_HOST_XFER=$1 SOFTMPM_XFER_DIRECT=$2 timeout 300 python bench.py --config c3 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('xfer=$1 direct=$2', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
  done
done
