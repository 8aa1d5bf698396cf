L=paper_2402_01181_b200
for r in 1 2; do
ROUNDS=1 bash tools/sweeps/ab.sh base=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
SOFTMPM_GRIDOP_SIMPLE=1 ROUNDS=1 bash tools/sweeps/ab.sh simple4=$L/libsoftmpm_b200.so simple2=$L/libsoftmpm_b200_gs2.so 2>&1 | grep -v '^ \|Trace\|json'
done
SOFTMPM_GRIDOP_SIMPLE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenes.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
