mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_run.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches_c3.csv > gpurun_out/r02_launches_c3.txt
head -25 gpurun_out/r02_launches_c3.txt
