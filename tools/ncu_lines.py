"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python tools/ncu_lines.py s.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur_file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))
    key = (cur_file, int(r[0]))
    src[key] = r[1].strip()[:80]
    for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed", "stall_long_sb",
              "stall_short_sb", "stall_barrier", "stall_mio", "stall_wait"):
        try:
            agg[key][k] += float(d.get(k, "0") or 0)
        except ValueError:
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
print(f"{'file:line':28s} {'stall%':>7s} {'instrs':>10s} long  short barr mio  | source")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    s = v["Warp Stall Sampling (All Samples)"]
    print(f"{key[0]+':'+str(key[1]):28s} {100*s/tot:6.1f}% {int(v['Instructions Executed']):10d} "
          f"{int(v['stall_long_sb']):4d} {int(v['stall_short_sb']):5d} {int(v['stall_barrier']):4d} "
          f"{int(v['stall_mio']):4d} | {src[key]}")
