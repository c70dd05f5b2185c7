"""Aggregate an ncu 'cuda,sass' source-page CSV by CUDA source line:
stall samples and executed warp instructions per line (top N).
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines_ls.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        if r[0] == "Line No":
            hdr = r
        continue
    if r[0] != "" and len(r) > 8:
        try:
            smp = float(r[4]); ins = float(r[7])
        except ValueError:
            continue
        agg.append((smp, ins, fname, r[0], r[1].strip()))
ts = sum(a[0] for a in agg) or 1; ti = sum(a[1] for a in agg) or 1
print("total samples %d, warp inst %.3e" % (ts, ti))
for smp, ins, f, ln, src in sorted(agg, key=lambda a: -a[0])[:N]:
    print("%5.1f%% smp %5.1f%% ins %s:%s  %s" % (100 * smp / ts, 100 * ins / ti, f, ln, src[:90]))
