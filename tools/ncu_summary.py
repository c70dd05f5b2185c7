"""Summarise ncu evidence into profiles/: per-kernel duration, DRAM traffic,
occupancy, issue activity, stall mix (full-set report) and the launch list.

    python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out-prefix>
"""
import csv, io, json, subprocess, sys
from collections import defaultdict

rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "warp_inst",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio": "ld_bytes_per_sector",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_mem_pct",
}
out = []
for r in data:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    rec = {"kernel": d.get("Kernel Name", "").split("(")[0]}
    for k, name in want.items():
        v = d.get(k)
        if v is None:
            continue
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        unit = u.get(k, "")
        if name == "duration":
            x = x * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
            rec["duration_ms"] = x
        elif name in ("dram_read", "dram_write"):
            x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            rec[name + "_bytes"] = x
        else:
            rec[name] = x
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0))
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and v not in ("", "n/a")]
    tot = sum(x for _, x in st) or 1
    rec["stalls"] = {k: round(100 * x / tot, 1) for k, x in sorted(st, key=lambda t: -t[1])[:5]}
    out.append(rec)

rows = list(csv.reader(open(launches))) if launches != "-" else [["Kernel Name", "Metric Value"]]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ui = h.index("Metric Unit") if "Metric Unit" in h else None
per = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "ns"
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        per[r[ki].split("(")[0]].append(v)

md = ["| kernel | launches | mean ms (ncu, cold, serialised) | max ms |", "|---|---|---|---|"] if per else []
for k, v in per.items():
    md.append(f"| {k} | {len(v)} | {sum(v)/len(v):.4f} | {max(v):.4f} |")
md.append("")
md.append("| kernel (full set) | ms | DRAM read MB | DRAM write MB | DRAM % peak | global ld B/sector (of 32) | L2 hit % | tensor pipe % | occupancy % | issue active % | regs | warp inst | top stalls (% of samples) |")
md.append("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
traffic = {}
for r in out:
    rd, wr = r.get("dram_read_bytes", 0), r.get("dram_write_bytes", 0)
    traffic[r["kernel"]] = rd + wr
    md.append(f"| {r['kernel']} | {r.get('duration_ms', 0):.3f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {r.get('dram_pct', 0):.1f} | "
              f"{r.get('ld_bytes_per_sector', 0):.1f} | {r.get('l2_hit_pct', 0):.1f} | {r.get('tensor_pipe_pct', 0):.1f} | "
              f"{r.get('occupancy_pct', 0):.1f} | {r.get('issue_active_pct', 0):.1f} | {int(r.get('regs', 0))} | "
              f"{int(r.get('warp_inst', 0))} | " + ", ".join(f"{k} {v}" for k, v in r["stalls"].items()) + " |")
open(prefix + "_ncu_summary.md", "w").write("\n".join(md) + "\n")
json.dump({"kernels": out, "dram_bytes_per_launch": traffic, "bytes_per_step": sum(traffic.values())},
          open(prefix + "_ncu.json", "w"), indent=1)
print("\n".join(md))
