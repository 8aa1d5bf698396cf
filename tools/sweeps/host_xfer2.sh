for d in 0 1; do SOFTMPM_XFER_DIRECT=$d timeout 300 python tools/probes/xfer_probe.py 1000000 2>&1 | grep "host_xfer=1" | sed "s/^/direct=$d /"; done
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_reference_cases.py tests/test_gpu_frame.py 2>&1 | tail -1
for r in 1 2; do
  for d in 0 1; do
    SOFTMPM_XFER_DIRECT=$d timeout 300 python bench.py --config c3 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('direct=$d', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), 'ms', round(d['ms_per_step'],3))"
  done
done
