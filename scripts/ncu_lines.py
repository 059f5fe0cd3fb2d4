#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of one ncu report
(ncu --page source --print-source cuda,sass), normalised per `unit` warps.

    python scripts/ncu_lines.py gpurun_out/prof_x.ncu-rep [units] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, cur, line = {}, None, None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        line = (cur, r[0], r[1].strip()[:90])
        continue
    try:
        n = int(r[7]) if r[7] not in ("", "-") else 0
        s = int(r[4]) if r[4] not in ("", "-") else 0
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(line, [0, 0])
    a[0] += n
    a[1] += s
tot = sum(v[0] for v in agg.values())
st = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot} ({tot / units:.1f} per unit)")
for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{n / units:8.1f} {100 * s / st:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
