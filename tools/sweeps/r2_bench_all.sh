# round-2 bench lines: default (C3, with CPU baselines incl. the numba reference), reference arm, C4, C5, N=2 plumbing
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/r02_bench_reference_arm.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_c3.err; echo "c3 rc=$?"; tail -c 300 gpurun_out/r02_bench_c3.json
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_c5.err; echo "c5 rc=$?"
SOFTMPM_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_n2_shared.json 2> gpurun_out/r02_n2.err; echo "n2 rc=$?"
