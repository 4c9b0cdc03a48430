"""Per-source-line and per-region dynamic instruction counts of the event-loop
kernel from an ncu source page exported with --print-source cuda,sass.
Usage: ncu_lines.py page.csv decisions [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
ndec = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur, agg = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "" and len(r) > 8:
        try:
            agg.append((cur, int(r[0]), r[1].strip()[:90], int(r[7] or 0), int(r[4] or 0), int(r[8] or 0)))
        except ValueError:
            pass
tot = sum(a[3] for a in agg)
ts = sum(a[4] for a in agg) or 1
print(f"warp instructions per decision {tot / ndec:.1f}")
for a in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{a[0][:14]:14} {a[1]:4} {a[3] / ndec:6.2f}/dec s{a[4] / ts * 100:4.1f}% t{a[5] / max(a[3], 1):4.1f} | {a[2]}")
