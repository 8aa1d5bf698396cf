for t in 8 12 16; do echo "threads $t"; SOFTMPM_HOST_THREADS=$t timeout 300 python tools/probes/xfer_probe.py 1000000 2>&1 | grep pageable; done
timeout 1500 python -m pytest -x -q tests/test_gpu_reference_suite.py tests/test_gpu_parity.py tests/test_gpu_reference_cases.py 2>&1 | tail -2
