for t in 16 8 4; do echo "threads $t"; SOFTMPM_HOST_THREADS=$t timeout 300 python tools/probes/xfer_probe.py 2>&1 | tail -6; done
