L=paper_2402_01181_b200
for r in 1 2; do
for k in 1 2 3; do SOFTMPM_REBIN_FRAMES=$k ROUNDS=1 bash tools/sweeps/ab.sh rf$k=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'; done
done
for c in c4 c5; do for k in 1 2; do SOFTMPM_REBIN_FRAMES=$k CONFIG=$c ROUNDS=1 STEPS=6 bash tools/sweeps/ab.sh ${c}_rf$k=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenes.py tests/test_gpu_fullsize.py -q --timeout 600 2>&1 | tail -2
