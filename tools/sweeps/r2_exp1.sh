ROUNDS=2 bash tools/sweeps/ab.sh base=paper_2402_01181_b200/libsoftmpm_b200.so freeze=paper_2402_01181_b200/libsoftmpm_b200_xfreeze.so noconf=paper_2402_01181_b200/libsoftmpm_b200_xnoconf.so sts=paper_2402_01181_b200/libsoftmpm_b200_xsts.so noscat=paper_2402_01181_b200/libsoftmpm_b200_xnoscat.so
SOFTMPM_LIB=paper_2402_01181_b200/libsoftmpm_b200_prof.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "^\[" 
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 60 -c 1 -o gpurun_out/r2_pk1_fused python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1
echo ncu rc $?
