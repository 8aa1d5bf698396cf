B3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B3 > gpurun_out/plain_c3b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv --log-file gpurun_out/r02_launches_c3_final.csv $B3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grid_op_simple -s 60 -c 1 -o gpurun_out/r02_gridop_c3 $B3 > gpurun_out/ncu_g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 60 -c 1 -o gpurun_out/r02_fused_c3_final $B3 > gpurun_out/ncu_f.log 2>&1
echo "rc=$?"
