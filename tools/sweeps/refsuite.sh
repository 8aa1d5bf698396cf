timeout 1200 python -m pytest -x -q tests/test_gpu_reference_suite.py tests/test_gpu_reference_demos.py 2>&1 | grep -E "unexpected|passed|failed|FAILED" | head -20
SOFTMPM_HOST_THREADS=12 timeout 300 python tools/probes/xfer_probe.py 2>&1 | tail -5
