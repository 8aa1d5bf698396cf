timeout 1300 python -m pytest tests/test_gpu_reference_suite.py -x -q -s --timeout 1250 > gpurun_out/ref_suite.log 2>&1; echo "ref suite rc=$?"; grep -E "passed|failed" gpurun_out/ref_suite.log | tail -3
ROUNDS=1 bash tools/sweeps/ab.sh base=paper_2402_01181_b200/libsoftmpm_b200.so one_cta=paper_2402_01181_b200/libsoftmpm_b200_x1cta.so 2>&1 | grep -v '^ \|Trace\|json'
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/r02_pytest_gpu.log
