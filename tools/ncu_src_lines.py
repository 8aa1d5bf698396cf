"""Per-CUDA-source-line instruction totals (and SASS opcode mix) from an ncu
source page exported with --print-source cuda,sass.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python tools/ncu_src_lines.py s.csv [top] [particles]
"""
import csv
import sys
from collections import defaultdict, Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
npart = float(sys.argv[3]) if len(sys.argv) > 3 else 0
cur_file, hdr, key = None, None, None
line_inst = defaultdict(float)
line_stall = defaultdict(float)
line_src = {}
line_ops = defaultdict(Counter)
op_tot = Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    d = dict(zip(hdr, r))
    if r[0].isdigit():
        key = (cur_file, int(r[0]))
        line_src[key] = r[1].strip()[:70]
        try:
            line_inst[key] += float(r[7] or 0)
            line_stall[key] += float(r[4] or 0)
        except ValueError:
            pass
    elif key is not None and len(r) > 7 and r[2].startswith("0x"):
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        op = op.split(".")[0]
        try:
            n = float(r[7] or 0)
        except ValueError:
            continue
        line_ops[key][op] += n
        op_tot[op] += n
tot = sum(line_inst.values())
stot = sum(line_stall.values()) or 1
scale = 32.0 / npart if npart else 1.0
print(f"total warp instructions {tot:.0f}" + (f"  = {tot*scale:.0f} thread-instr/particle" if npart else ""))
print("opcodes:", ", ".join(f"{k} {v*scale:.0f}" for k, v in op_tot.most_common(18)))
for key, v in sorted(line_inst.items(), key=lambda kv: -kv[1])[:top]:
    ops = " ".join(f"{k}:{c*scale:.0f}" for k, c in line_ops[key].most_common(4))
    print(f"{key[0]+':'+str(key[1]):22s} {v*scale:8.1f} {100*line_stall[key]/stot:5.1f}%  {line_src[key][:60]:60s} {ops}")
