# round-2 evidence: surface parity tests, then per-config ncu captures of the
# fused kernel (full set, warm-cache DRAM, launch list) for c3 and c5
timeout 900 python -m pytest tests/test_gpu_surface.py -q --timeout 600 > gpurun_out/surface.log 2>&1; echo "surface rc=$?"; tail -2 gpurun_out/surface.log
B3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 60 -c 1 -o gpurun_out/r02_fused_c3 $B3 > gpurun_out/ncu_c3.log 2>&1 && \
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fused_kernel -s 60 -c 12 --csv --log-file gpurun_out/r02_warm_c3.csv $B3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv --log-file gpurun_out/r02_launches_c3.csv $B3 > /dev/null 2>&1
echo "c3 ncu rc=$?"
B5="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline"
$B5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 40 -c 1 -o gpurun_out/r02_fused_c5 $B5 > gpurun_out/ncu_c5.log 2>&1 && \
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fused_kernel -s 40 -c 6 --csv --log-file gpurun_out/r02_warm_c5.csv $B5 > /dev/null 2>&1
echo "c5 ncu rc=$?"
