# Host-converted transfers: parity subset, then e2e A/B (SOFTMPM_HOST_XFER=0 / 1) at C3.
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_reference_cases.py tests/test_gpu_frame.py tests/test_gpu_scenes.py tests/test_gpu_slab.py 2>&1 | tail -2
for r in 1 2; do
  for v in 0 1; do
    SOFTMPM_HOST_XFER=$v timeout 300 python bench.py --config c3 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('xfer=$v', 'value', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), 'ms', round(d['ms_per_step'],3))"
  done
done
