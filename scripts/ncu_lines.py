"""Per-source-line stall samples / executed instructions from
`ncu -i REP --page source --csv --print-source cuda,sass` output (stdin)."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
agg, src, cur = {}, {}, None
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    if cur is None:
        continue
    try:
        s, ie = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += s
    a[1] += ie
tot = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{k[0][:14]:14s}:{k[1]:<4d} {100*a[0]/tot:5.1f}% stall {100*a[1]/ti:5.1f}% inst  {src[k][:80]}")
