mkdir -p gpurun_out
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fused_kernel --launch-skip 60 --launch-count 20 --csv --log-file gpurun_out/warm_dram_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py warm gpurun_out/warm_dram_c3.csv
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/warm_dram_c3.csv')) if len(r)>10]
h=rows[0]; mi,vi=h.index("Metric Name"),h.index("Metric Value")
acc=collections.defaultdict(list)
for r in rows[1:]: acc[r[mi]].append(float(r[vi].replace(',','')))
for k,v in acc.items(): print(k, [round(x/1e6,1) if 'bytes' in k else round(x/1e3,1) for x in v])
PY
