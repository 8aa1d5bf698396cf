# Whole GPU suite + xfer probe.
timeout 2400 python -m pytest -x -q -m gpu tests 2>&1 | tail -6
SOFTMPM_HOST_THREADS=12 timeout 300 python tools/probes/xfer_probe.py 2>&1 | tail -6
