"""Summarise an ncu report's source page: per CUDA line warp-stall samples and
instructions executed (needs -lineinfo).  Usage: ncu_lines.py report.ncu-rep [kernel-regex] [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if kern:
    cmd += ["-k", "regex:" + kern]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit() or len(r) < 8:
        continue
    try:
        samp = int(r[4]); inst = int(r[7])
    except ValueError:
        continue
    out.append((samp, inst, cur, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out)
print(f"total stall samples {tot}  total warp instructions {ti}")
for o in sorted(out, reverse=True)[:N]:
    print(f"{o[0]:7d} {100*o[0]/tot:5.1f}%  inst {o[1]:11d}  {o[2]}:{o[3]}  {o[4]}")
