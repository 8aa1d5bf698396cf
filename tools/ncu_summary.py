"""Summaries of ncu captures for profiles/ (run here, on the .ncu-rep files gpurun brings back).

usage:
  python tools/ncu_summary.py full   X.ncu-rep  > profiles/rNN_ncu_<kernel>.json
      one `ncu --set full` capture: duration, DRAM bytes (the bench's
      roofline "traffic"), issue/occupancy, stall breakdown, shared-memory
      wavefronts, executed instructions by SASS opcode
  python tools/ncu_summary.py launches L.csv > profiles/rNN_launches.txt
      a `--metrics gpu__time_duration.sum --csv --log-file L.csv` launch list:
      per-kernel count / total / mean and share of all kernel time
"""
import collections
import csv
import json
import subprocess
import sys


def _f(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): _f(v) for k, v in d.items()
                  if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and _f(v) is not None}
        tot = sum(stalls.values()) or 1.0
        rd, wr = _f(d.get("dram__bytes_read.sum")), _f(d.get("dram__bytes_write.sum"))
        units = dict(zip(hdr, rows[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get("dram__bytes_read.sum", ""), 1e6)
        tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6}.get(
            units.get("gpu__time_duration.sum", ""), 1.0)
        dur = _f(d.get("gpu__time_duration.sum"))
        rec = {
            "kernel": d.get("Kernel Name"),
            "duration_us": dur * tscale if dur is not None else None,
            "dram_read_bytes": rd * scale if rd is not None else None,
            "dram_write_bytes": wr * scale if wr is not None else None,
            "issue_active_pct": _f(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active")),
            "warps_active_pct": _f(d.get("sm__warps_active.avg.pct_of_peak_sustained_active")),
            "registers_per_thread": _f(d.get("launch__registers_per_thread")),
            "grid_size": _f(d.get("launch__grid_size")),
            "block_size": _f(d.get("launch__block_size")),
            "inst_executed": _f(d.get("smsp__inst_executed.sum")),
            "l2_hit_pct": _f(d.get("lts__t_sector_hit_rate.pct")),
            "smem_wavefronts": _f(d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")),
            "smem_bank_conflicts": _f(d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")),
            "stall_pct": {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])
                          if 100 * v / tot >= 0.5},
        }
        if rec["dram_read_bytes"] is not None and rec["dram_write_bytes"] is not None:
            rec["dram_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        out.append(rec)
    # executed instructions by opcode (SASS source page)
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    ops = collections.Counter()
    h = None
    for r in csv.reader(sass.splitlines()):
        if not r:
            continue
        if len(r) > 1 and r[1] == "Source":
            h = r
            continue
        if h is None:
            continue
        d = dict(zip(h, r))
        n = _f(d.get("Instructions Executed", ""))
        toks = d.get("Source", "").split()
        if n is None or not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[op.split(".")[0]] += n
    if out and ops:
        tot = sum(ops.values())
        out[0]["inst_by_opcode_pct"] = {k: round(100 * v / tot, 1) for k, v in ops.most_common(16)}
    json.dump(out if len(out) > 1 else out[0], sys.stdout, indent=1)
    print()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        v = _f(r[vi]) or 0.0
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"{'kernel':56s} {'launches':>8s} {'total us':>11s} {'mean us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:56]:56s} {n:8d} {t / 1e3:11.1f} {t / n / 1e3:9.2f} {100 * t / tot:5.1f}%")
    print(f"{'all':56s} {sum(a[0] for a in agg.values()):8d} {tot / 1e3:11.1f}")


def warm(csv_path):
    """Mean DRAM bytes per launch of each kernel in a warm-cache, no-replay
    capture (`ncu --cache-control none --metrics dram__bytes_read.sum,
    dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file W.csv`)."""
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    acc = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
                 "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        v = _f(r[vi])
        if v is not None:
            acc[r[ki]][r[mi]].append(v * scale)
    out = {}
    for k, m in acc.items():
        rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
        out[k] = {"launches": len(rd), "dram_bytes_warm": (sum(rd) + sum(wr)) / max(len(rd), 1),
                  "duration_us_warm": sum(m.get("gpu__time_duration.sum", [])) / max(len(rd), 1)}
    return out


if __name__ == "__main__":
    if sys.argv[1] == "full" and "--warm" in sys.argv:
        # full X.ncu-rep --warm W.csv --config cN: one record with the warm DRAM bytes merged in
        import io
        from contextlib import redirect_stdout
        buf = io.StringIO()
        with redirect_stdout(buf):
            full(sys.argv[2])
        recs = json.loads(buf.getvalue())
        recs = recs if isinstance(recs, list) else [recs]
        w = warm(sys.argv[sys.argv.index("--warm") + 1])
        cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
        for rec in recs:
            hit = [v for k, v in w.items() if k.split("(")[0].strip() in str(rec.get("kernel"))]
            if hit:
                rec.update(hit[0])
            if cfg:
                rec["config"] = cfg
        print(json.dumps(recs[0] if len(recs) == 1 else recs, indent=1))
    else:
        {"full": full, "launches": launches, "warm": lambda p: print(json.dumps(warm(p), indent=1))}[sys.argv[1]](sys.argv[2])
