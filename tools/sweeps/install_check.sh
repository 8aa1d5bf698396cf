timeout 1500 python -m pytest -x -q tests/test_gpu_reference_suite.py tests/test_gpu_reference_demos.py tests/test_gpu_scenes.py 2>&1 | tail -2
timeout 900 python tools/probes/ref_cli_bench.py 2>&1 | tail -4
